import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, crdata, oracle
from oracle import ref
import paper_1608_02227_b200 as crp
N, n = int(sys.argv[1]), int(sys.argv[2])
X, ybar = crdata.paper_problem(N, n, "quad")
g = 1e-4
L = ref.lipschitz(X, g)
o = oracle.papg_adaptive(X, ybar, g, L, 60)
for mode in ("step", "solve", "solve_stop"):
    s = crp.Solver(X, ybar, g, L=L, prec="fp64", adaptive=True)
    s.set_step_rule("adaptive", 2.0)
    tr = []
    if mode == "step":
        for _ in range(60):
            s.step(); tr.append(s.step_info()["trials_last"])
    elif mode == "solve":
        for _ in range(60):
            s.solve(1); tr.append(s.step_info()["trials_last"])
    else:
        for _ in range(12):
            s.solve(5, report_every=5, infeas_tol=0.0, gap_tol=0.0); tr.append(s.step_info()["trials_last"])
    T = s.get_theta()[0]
    print(mode, "trials", tr[:30], "relT %.3e" % (np.linalg.norm(T - o["Tprev"]) / np.linalg.norm(o["Tprev"])), s.step_info())
print("oracle trials", list(o["trials"][:30]), o["s"] / L)
