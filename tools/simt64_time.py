"""Time the fp64 CUDA-core pass (kernel='simt', prec='fp64') on a C3-shaped problem.

    python tools/simt64_time.py [N] [n] [iters]
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 4000
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    it = int(sys.argv[3]) if len(sys.argv) > 3 else 50
    import torch
    import crdata
    import paper_1608_02227_b200 as crp
    X, ybar = crdata.random_problem(N, n, seed=0, law="uniform")
    for prec in ("fp64", "fp32"):
        s = crp.Solver(X, ybar, 1e-3, prec=prec, kernel="simt")
        s.solve(10)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        s.solve(it)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / it
        print(f"simt {prec} N={N} n={n}: {ms * 1e3:.1f} us/iteration, {N * N / (ms * 1e-3):.3e} pairs/s")
        s.close()


if __name__ == "__main__":
    main()
