"""Build libsrsb.so in-tree for sm_100a (parallel nvcc per translation unit, then link).

    python -m paper_2003_12693_b200.build [--force] [-j N]
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(CSRC, "build")
LIB = os.path.join(HERE, "libsrsb.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
def _nccl_dir():
    """NCCL 2.28 shipped with the torch wheel (nvidia-nccl): headers + libnccl.so.2."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations if spec else []):
        d = os.path.join(base, "nccl")
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return d
    raise RuntimeError("nccl.h not found (nvidia-nccl wheel)")


NCCL = _nccl_dir()
FLAGS = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-I", INCLUDE, "-I", os.path.join(NCCL, "include"),
         "-Xptxas", "-v", "--expt-relaxed-constexpr"] + os.environ.get("SRSB_NVCC_FLAGS", "").split()
LDFLAGS = ["-L", os.path.join(NCCL, "lib"), "-l:libnccl.so.2", "-Xlinker", "-rpath=" + os.path.join(NCCL, "lib")]


def _deps():
    return sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) +
                  glob.glob(os.path.join(INCLUDE, "*.h")))


_INC = None


def _src_deps(path: str, seen=None) -> set:
    """Headers a source reaches through #include "..." (resolved in csrc/ and include/), recursively."""
    import re
    seen = set() if seen is None else seen
    for m in re.finditer(r'^\s*#\s*include\s+"([^"]+)"', open(path).read(), re.M):
        for base in (os.path.dirname(path), CSRC, INCLUDE):
            q = os.path.normpath(os.path.join(base, m.group(1)))
            if os.path.exists(q):
                if q not in seen:
                    seen.add(q)
                    _src_deps(q, seen)
                break
    return seen


def _compile(src: str, force: bool) -> tuple[str, str]:
    obj = os.path.join(OBJ, os.path.basename(src).replace(".cu", ".o"))
    log = obj + ".ptxas.log"
    stamp = obj + ".flags"
    flags = " ".join(ARCH + FLAGS)
    newest = max(os.path.getmtime(p) for p in [src] + sorted(_src_deps(src)))
    same_flags = os.path.exists(stamp) and open(stamp).read() == flags
    if not force and same_flags and os.path.exists(obj) and os.path.getmtime(obj) >= newest:
        return obj, "cached"
    cmd = [NVCC] + ARCH + FLAGS + ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    with open(log, "w") as f:
        f.write(r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr[-4000:]}")
    with open(stamp, "w") as f:
        f.write(flags)
    return obj, "built"


LIB_STAMP = LIB + ".flags"


def _up_to_date() -> bool:
    """The .so is newer than every source/header and was linked with the current flags."""
    if not (os.path.exists(LIB) and os.path.exists(LIB_STAMP)):
        return False
    if open(LIB_STAMP).read() != " ".join(ARCH + FLAGS + LDFLAGS):
        return False
    newest = max(os.path.getmtime(p) for p in glob.glob(os.path.join(CSRC, "*.cu")) + _deps())
    return os.path.getmtime(LIB) >= newest


def build(force: bool = False, jobs: int | None = None, verbose: bool = False) -> str:
    if not force and _up_to_date():
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    jobs = jobs or max(1, os.cpu_count() or 1)
    with cf.ThreadPoolExecutor(jobs) as ex:
        results = list(ex.map(lambda s: _compile(s, force), srcs))
    objs = [o for o, _ in results]
    relink = force or not os.path.exists(LIB) or any(st == "built" for _, st in results) or \
        os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs)
    if relink:
        tmp = LIB + ".tmp"
        cmd = [NVCC] + ARCH + ["-shared", "-o", tmp] + objs + ["-lcudart"] + LDFLAGS
        subprocess.check_call(cmd)
        os.replace(tmp, LIB)
        with open(LIB_STAMP, "w") as f:
            f.write(" ".join(ARCH + FLAGS + LDFLAGS))
    if verbose:
        for s, (_, st) in zip(srcs, results):
            print(f"{os.path.basename(s)}: {st}")
    return LIB


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-j", type=int, default=None)
    a = ap.parse_args(argv)
    print(build(force=a.force, jobs=a.j, verbose=True))


if __name__ == "__main__":
    sys.exit(main())
