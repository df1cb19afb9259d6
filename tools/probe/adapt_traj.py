import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, crdata
import paper_1608_02227_b200 as crp
N, n, f0 = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
X, ybar = crdata.paper_problem(N, n, f0)
g = 1e-4
s = crp.Solver(X, ybar, g, prec="fp64" if n <= 24 else "fp32", adaptive=True)
L = s.L
s.set_step_rule("adaptive", 2.0)
for k in range(40):
    st = s.solve(250, report_every=250, infeas_tol=0, gap_tol=0)["last"]
    info = s.step_info()
    print((k + 1) * 250, "s/L %.3g" % (info["s"] / L), "trials %d" % info["trials_total"], "infeas %.3g" % st["infeas_norm"],
          "gap %.3g" % (abs(st["gap"]) / (N * N - N)), "g %.8g" % st["g"], "r %.8g" % st["r_gamma"], flush=True)
