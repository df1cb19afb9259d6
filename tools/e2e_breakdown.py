"""Where the end-to-end time of bench.py's e2e leg goes (C4 by default)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import crdata
import paper_1608_02227_b200 as crp
cfg = crdata.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
K = int(sys.argv[2]) if len(sys.argv) > 2 else 200
X, ybar = crdata.make_problem(cfg)
Xp = torch.from_numpy(X).pin_memory().numpy(); yp = torch.from_numpy(ybar).pin_memory().numpy()
crp.Solver(X[:300], ybar[:300], cfg.gamma).close()     # warm the library / context
torch.cuda.synchronize()
t0 = time.perf_counter()
L = crp.lipschitz_host(Xp, cfg.gamma) if os.environ.get("HOST_L") else 0.0
t1 = time.perf_counter()
s = crp.Solver(Xp, yp, cfg.gamma, L=L, prec=cfg.prec)     # L = 0: device Lanczos inside cr_init
torch.cuda.synchronize(); t2 = time.perf_counter()
s.solve(K); torch.cuda.synchronize(); t3 = time.perf_counter()
y, xi, st = s.primal(); t4 = time.perf_counter()
print(f"{cfg.name}: host lanczos {1e3*(t1-t0):.1f} ms, init (alloc+H2D+setup[+device L]) {1e3*(t2-t1):.1f} ms, L={s.L:.6e}, "
      f"solve({K}) {1e3*(t3-t2):.1f} ms ({1e3*(t3-t2)/K:.3f} ms/it), primal {1e3*(t4-t3):.1f} ms")
