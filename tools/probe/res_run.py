import os, sys
sys.path.insert(0, os.getcwd())
import crdata, paper_1608_02227_b200 as crp
c = crdata.CONFIGS[sys.argv[1]]
X, ybar = crdata.make_problem(c)
s = crp.Solver(X, ybar, c.gamma, prec=c.prec)
s.solve(int(sys.argv[2]))
s.stream.synchronize()
print("ok")
