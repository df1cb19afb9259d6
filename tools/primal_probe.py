"""cr_primal timing at a config: repeated calls in one process, first call separated (lazy module
loading / first-launch costs) from the steady state.  Usage: primal_probe.py [C4] [reps]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import crdata
import paper_1608_02227_b200 as crp
cfg = crdata.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
X, ybar = crdata.make_problem(cfg)
print("CUDA_MODULE_LOADING =", os.environ.get("CUDA_MODULE_LOADING"), flush=True)
for trial in range(2):
    s = crp.Solver(X, ybar, cfg.gamma, prec=cfg.prec)
    s.solve(20)
    torch.cuda.synchronize()
    ts = []
    yo = torch.empty(cfg.N, dtype=torch.float64).pin_memory().numpy()
    xo = torch.empty((cfg.N, cfg.n), dtype=torch.float64).pin_memory().numpy()
    for r in range(reps):
        t0 = time.perf_counter()
        y, xi, st = s.primal(out=(yo, xo))
        ts.append(1e3 * (time.perf_counter() - t0))
    print(f"{cfg.name} solver {trial}: primal ms " + " ".join(f"{t:.2f}" for t in ts), flush=True)
    s.close()
