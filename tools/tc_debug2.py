import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import crdata
import paper_1608_02227_b200 as crp
N, n = int(sys.argv[1]), int(sys.argv[2])
X, ybar = crdata.random_problem(N, n, seed=5, fp32=True)
np.set_printoptions(precision=5, linewidth=200)
s = crp.Solver(X, ybar, 1e-3, kernel="tc")
s.step(); s.step()
T = s.get_theta()[0]
r, c, P = s.get_sums(0)
print("dbg", os.environ.get("CR_TC_DEBUG"), "r[:6]", r[:6], "P[0,:6]", P[0, :6])
print("   rowsum T", T.sum(1)[:6], " colsum X (per tile sums)", X[:32].sum(0)[:4], X.sum(0)[:4])
