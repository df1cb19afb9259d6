"""One cr_primal at a config (ncu target for the fp64 residual pass)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import crdata
import paper_1608_02227_b200 as crp
cfg = crdata.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C5"]
X, ybar = crdata.make_problem(cfg)
s = crp.Solver(X, ybar, cfg.gamma, prec=cfg.prec)
s.solve(3)
torch.cuda.synchronize()
t0 = time.perf_counter()
y, xi, st = s.primal()
print(f"{cfg.name} primal {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
