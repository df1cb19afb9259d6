import os, sys, json
sys.path.insert(0, os.getcwd())
import numpy as np, crdata
from oracle import ref
import paper_1608_02227_b200 as crp
N, n = 2400, 20
X, ybar = crdata.paper_problem(N, n, "quad")
g = 1e-4
L = ref.lipschitz(X, g)
s = crp.Solver(X, ybar, g, L=L, prec="fp64", adaptive=True)
s.set_step_rule("adaptive", 2.0)
tr = []
for chunk in range(10):
    for _ in range(25):
        s.step(); tr.append(s.step_info()["trials_last"])
    st = s.primal()[2]
    print((chunk + 1) * 25, "s/L %.3g" % (s.step_info()["s"] / L), "infeas %.3g" % st["infeas_norm"], "g %.8g" % st["g"], flush=True)
json.dump(tr, open("gpurun_out/gpu_trials_2400.json", "w"))
