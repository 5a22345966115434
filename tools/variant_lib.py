"""Link a tuning variant of libsrsb.so: recompile a few translation units with extra nvcc flags
(e.g. -DSRSB_C2R_MINB=3) and link them with the current objects of the main build.

    python tools/variant_lib.py NAME "FLAGS" fft_c2r.cu [more.cu ...]   ->  vlib/libsrsb_NAME.so

Load it with SRSB_LIB=vlib/libsrsb_NAME.so (paper_2003_12693_b200/srsb.py).  Measurement aid only.
"""
import glob
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2003_12693_b200 import build as B  # noqa: E402


def main(name, flags, srcs):
    B.build()
    out_dir = os.path.join(os.path.dirname(B.HERE), "vlib")
    os.makedirs(os.path.join(out_dir, name), exist_ok=True)
    objs = {os.path.basename(o): o for o in glob.glob(os.path.join(B.OBJ, "*.o"))}
    for s in srcs:
        o = os.path.join(out_dir, name, s.replace(".cu", ".o"))
        subprocess.check_call([B.NVCC] + B.ARCH + B.FLAGS + flags.split() + ["-c", os.path.join(B.CSRC, s), "-o", o],
                              stdout=subprocess.DEVNULL)
        objs[os.path.basename(o)] = o
    lib = os.path.join(out_dir, f"libsrsb_{name}.so")
    subprocess.check_call([B.NVCC] + B.ARCH + ["-shared", "-o", lib] + sorted(objs.values()) + ["-lcudart"] + B.LDFLAGS)
    print(lib)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3:])
