"""Context run on the paper's own Section 4 workload (crdata.paper_problem): time to
the paper's stopping rule (normalized infeasibility <= 1e-1 and |theta^T C eta|/(N^2-N) <= 5e-7,
P:1106) with gamma = 1e-4, constant and adaptive steps, on one B200.  The paper's wall times
(MATLAB + MOSEK, K = N/100 blocks, 24-core node) are in BASELINE.md -- context, not a target:
the configurations (K = N here) and hardware differ.

    python tools/paper_workload.py 2400 20 quad
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import crdata  # noqa: E402
import paper_1608_02227_b200 as crp  # noqa: E402

N, n, f0 = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
cap = int(sys.argv[4]) if len(sys.argv) > 4 else 200000
X, ybar = crdata.paper_problem(N, n, f0)
prec = "fp64" if n <= 24 else "fp32"
out = {"N": N, "n": n, "f0": f0, "gamma": 1e-4, "prec": prec}
rules = os.environ.get("RULES", "constant,adaptive,backtrack").split(",")
for rule in rules:
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    # "partition": the paper's own configuration, K = N / 100 blocks, constant step
    nbar = 100 if rule == "partition" else 1
    s = crp.Solver(X, ybar, 1e-4, prec=prec, adaptive=rule in ("adaptive", "backtrack"), nbar=nbar)
    if rule == "adaptive":
        s.set_step_rule("adaptive", 2.0)
    elif rule == "backtrack":
        s.set_step_rule("backtrack", 2.0, s_prev=s.L / 64)
    rep = s.solve(cap, report_every=50, infeas_tol=1e-1, gap_tol=5e-7)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    last = rep["last"]
    out[rule] = {"seconds": dt, "iters": rep["iters"], "converged": rep["converged"],
                 "infeas_norm": last["infeas_norm"], "gap_norm": abs(last["gap"]) / (N * N - N),
                 "r_gamma": last["r_gamma"], "s_over_L": s.step_info()["s"] / s.L}
    if nbar > 1:
        out[rule]["partition_stats"] = s.partition_info(check=False)
    s.close()
print(json.dumps(out))
