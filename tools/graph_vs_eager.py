"""Step time with the constant-step CUDA graphs (pass timing off) vs eager launches with the
per-pass events bench.py records (pass timing on)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import crdata
import paper_1608_02227_b200 as crp
cfg = crdata.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
K = int(sys.argv[2]) if len(sys.argv) > 2 else 300
X, ybar = crdata.make_problem(cfg)
s = crp.Solver(X, ybar, cfg.gamma, prec=cfg.prec)
s.solve(10)
for rep in range(2):
    for timing in (False, True):
        s.set_pass_timing(timing)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s.stream)
        s.solve(K)
        e1.record(s.stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / K
        extra = ""
        if timing:
            pm, pn = s.pass_timing()
            extra = f" pass avg {pm / max(pn, 1):.4f} ms"
        print(f"{cfg.name} timing={timing}: {ms:.4f} ms/step{extra}", flush=True)
        s.set_pass_timing(False)
