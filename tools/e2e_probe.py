"""Time the pieces of bench.py's e2e leg the way bench.py runs it (a first Solver alive)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import crdata
import paper_1608_02227_b200 as crp
cfg = crdata.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
K = int(sys.argv[2]) if len(sys.argv) > 2 else 100
X, ybar = crdata.make_problem(cfg)
s = crp.Solver(X, ybar, cfg.gamma, prec=cfg.prec)
s.solve(5)
torch.cuda.synchronize()
Xp = torch.from_numpy(X).pin_memory().numpy(); yp = torch.from_numpy(ybar).pin_memory().numpy()
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s2 = crp.Solver(Xp, yp, cfg.gamma, prec=cfg.prec)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    s2.solve(K); torch.cuda.synchronize(); t2 = time.perf_counter()
    y, xi, _ = s2.primal(); t3 = time.perf_counter()
    s2.close()
    print(f"{cfg.name} rep {rep}: init {1e3*(t1-t0):.1f} ms, solve({K}) {1e3*(t2-t1):.1f} ms, primal {1e3*(t3-t2):.1f} ms", flush=True)
