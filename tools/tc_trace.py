"""Debug: timeline of the tensor-core pass roles for CTA 0 (CR_TC_TRACE)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
path = "/tmp/tc_trace.bin"
os.environ["CR_TC_TRACE"] = path
import crdata
import paper_1608_02227_b200 as crp
X, ybar = crdata.make_problem(cfg)
s = crp.Solver(X, ybar, 1e-3, kernel="tc")
for _ in range(3):
    s.step()
t = np.fromfile(path, dtype=np.uint64).reshape(5, 256, 8).astype(np.int64)
t0 = t[t > 0].min()
t = np.where(t > 0, t - t0, -1)
names = ["prod", "mma", "store", "wg0", "wg1"]
for u in range(0, 24):
    row = []
    for r in range(5):
        ev = [v for v in t[r, u] if v >= 0]
        row.append(f"{names[r]}:" + ",".join(f"{v/1000:.1f}" for v in ev))
    print(u, " | ".join(row))
# per-tile period from the epilogue tile starts
for wg in (3, 4):
    st = t[wg, :, 0]; st = st[st >= 0]
    d = np.diff(st)
    print(names[wg], "tile period (kcycles) median", np.median(d) / 1000 if len(d) else None)
ev = t[3, 2:200:2]
ev = ev[(ev >= 0).all(axis=1)] if len(ev) else ev
if len(ev):
    seg = np.diff(ev[:, :7], axis=1)
    print("wg0 segment medians (kcycles): full-wait, d1-wait, at_empty-wait, compute, barrier, tail:",
          np.round(np.median(seg, axis=0) / 1000, 2))
m = t[1, 2:200]
m = m[(m[:, :6] >= 0).all(axis=1)]
if len(m):
    print("mma: gemm1 wait, gemm1 issue, (gap), at_full wait, gemm2 issue:",
          np.round(np.median(np.diff(m[:, :6], axis=1), axis=0) / 1000, 2))
