"""Build the CHECKED variant of libsrsb.so: every translation unit recompiled with -DSRSB_CHECKS
(shared-memory bounds assertions at the staged-access sites, sr_tma.cuh SRSB_CHK), linked to
vlib/libsrsb_checks.so.  Run the GPU tests against it with SRSB_LIB=vlib/libsrsb_checks.so.

    python tools/checked_lib.py
"""
import concurrent.futures as cf
import glob
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2003_12693_b200 import build as B  # noqa: E402


def main():
    out_dir = os.path.join(os.path.dirname(B.HERE), "vlib", "checks")
    os.makedirs(out_dir, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(B.CSRC, "*.cu")))
    flags = [f for f in B.FLAGS if f not in ("-Xptxas", "-v")] + ["-DSRSB_CHECKS"]

    def comp(src):
        o = os.path.join(out_dir, os.path.basename(src).replace(".cu", ".o"))
        subprocess.check_call([B.NVCC] + B.ARCH + flags + ["-c", src, "-o", o])
        return o
    with cf.ThreadPoolExecutor(os.cpu_count() or 4) as ex:
        objs = list(ex.map(comp, srcs))
    lib = os.path.join(os.path.dirname(out_dir), "libsrsb_checks.so")
    subprocess.check_call([B.NVCC] + B.ARCH + ["-shared", "-o", lib] + objs + ["-lcudart"] + B.LDFLAGS)
    print(lib)


if __name__ == "__main__":
    main()
