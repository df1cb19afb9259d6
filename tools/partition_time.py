"""Time the partition (K < N) path: ms per P-APG iteration and the block-projection share.
Usage: python tools/partition_time.py N n nbar [prec] [iters]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import crdata
import paper_1608_02227_b200 as crp

N, n, nbar = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
prec = sys.argv[4] if len(sys.argv) > 4 else "fp32"
iters = int(sys.argv[5]) if len(sys.argv) > 5 else 10
X, ybar = crdata.random_problem(N, n, seed=1, fp32=prec == "fp32")
out = {}
for nb in (1, nbar):
    s = crp.Solver(X, ybar, 1e-3, prec=prec, nbar=nb)
    s.solve(3)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s.stream)
    s.solve(iters)
    e1.record(s.stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / iters
    info = s.partition_info(check=False)
    y, xi, st = s.primal()
    out[nb] = ms
    print(f"N={N} n={n} nbar={nb} {prec}: {ms:.3f} ms/iter  {info} "
          f"max_violation={st['max_violation']:.3e} r_gamma={st['r_gamma']:.6e}", flush=True)
    s.close()
