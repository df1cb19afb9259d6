"""One cr_primal after a short solve (ncu target for the residual pass).  Usage: primal_once.py C4"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import crdata
import paper_1608_02227_b200 as crp
cfg = crdata.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
X, ybar = crdata.make_problem(cfg)
s = crp.Solver(X, ybar, cfg.gamma, prec=cfg.prec)
s.solve(3)
yo = torch.empty(cfg.N, dtype=torch.float64).pin_memory().numpy()
xo = torch.empty((cfg.N, cfg.n), dtype=torch.float64).pin_memory().numpy()
for _ in range(2):
    s.primal(out=(yo, xo))
torch.cuda.synchronize()
print("ok")
