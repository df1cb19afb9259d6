"""Debug: phase timeline (clock64, CTA 0) of the SMEM-resident solver (CR_TC_TRACE)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
path = "/tmp/rs_trace.bin"
os.environ["CR_TC_TRACE"] = path
import crdata
import paper_1608_02227_b200 as crp
c = crdata.CONFIGS[cfg]
X, ybar = crdata.make_problem(c)
s = crp.Solver(X, ybar, c.gamma, prec=c.prec)
s.solve(16)
t = np.fromfile(path, dtype=np.uint64).reshape(16, 8).astype(np.int64)
names = ["A", "sync1", "ycopy", "B1", "B2", "sync2", "C+"]
for it in range(2, 16, 3):
    d = np.diff(t[it, :7])
    nxt = t[it + 1, 0] - t[it, 6] if it + 1 < 16 else 0
    print(it, " ".join(f"{names[k]}={d[k]}" for k in range(6)), f"C={nxt}", "total", t[it + 1, 0] - t[it, 0] if it + 1 < 16 else "")
