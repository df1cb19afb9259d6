import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, crdata, paper_1608_02227_b200 as crp
cfg = sys.argv[1]; K = int(sys.argv[2]); timing = int(sys.argv[3])
X, ybar = crdata.make_problem(crdata.CONFIGS[cfg])
s = crp.Solver(X, ybar, 1e-3, kernel="tc")
s.set_pass_timing(bool(timing))
done = 0
try:
    while done < K:
        s.solve(100); done += 100
        s.stream.synchronize()
    print("ok", done)
except Exception as e:
    print("FAIL after", done, str(e)[:200])
