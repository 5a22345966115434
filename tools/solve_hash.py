"""sha256 of the phi-solve output (debug_solve) on a fixed seeded right-hand side: compare builds / variants bitwise.
    python tools/solve_hash.py M N [batch]        (SRSB_LIB selects the library)"""
import hashlib
import sys

import numpy as np
import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_2003_12693_b200 import Solver  # noqa: E402


def main():
    M, N = int(sys.argv[1]), int(sys.argv[2])
    B = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    F = torch.from_numpy(np.random.default_rng(5).standard_normal((B, M, N)).astype(np.float32)).cuda()
    with Solver(M, N, B, window=4) as sv:
        out = sv.debug_solve(F)
        torch.cuda.synchronize()
        print(hashlib.sha256(out.cpu().numpy().tobytes()).hexdigest())


if __name__ == "__main__":
    main()
