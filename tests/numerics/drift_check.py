"""Diagnostic: GPU (libcr) vs fp64 oracle drift of eta(Theta^K) diagnostics along a run.

    python tests/numerics/drift_check.py C2 500,1000,2000 [fp32|fp64] [simt|tc]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

import crdata  # noqa: E402
import oracle  # noqa: E402
from oracle import ref  # noqa: E402
import paper_1608_02227_b200 as crp  # noqa: E402

name = sys.argv[1]
ks = [int(v) for v in sys.argv[2].split(",")]
cfg = crdata.CONFIGS[name]
prec = sys.argv[3] if len(sys.argv) > 3 else cfg.prec
kernel = sys.argv[4] if len(sys.argv) > 4 else "auto"
N = int(os.environ.get("DRIFT_N", cfg.N))
X, ybar = crdata.make_problem(cfg, N=N)
L = ref.lipschitz(X, cfg.gamma)
s = crp.Solver(X, ybar, cfg.gamma, L=L, prec=prec, kernel=kernel)
o = None
done = 0
for K in ks:
    s.solve(K - done)
    o = oracle.papg(X, ybar, cfg.gamma, L, K - done, Tprev=None if o is None else o["Tprev"],
                    Tt=None if o is None else o["Tt"], t=1.0 if o is None else o["t"])
    done = K
    yo, xio = oracle.eta(X, ybar, cfg.gamma, o["Tprev"])
    so = oracle.stats(X, ybar, cfg.gamma, o["Tprev"], yo, xio)
    y, xi, sg = s.primal()
    T = s.get_theta()[0]
    out = {k: (so[k], abs(sg[k] - so[k]) / max(abs(so[k]), 1e-300)) for k in so}
    out["theta_rel"] = float(np.linalg.norm(T - o["Tprev"]) / np.linalg.norm(o["Tprev"]))
    out["y_rel"] = float(np.linalg.norm(y - yo) / np.linalg.norm(yo))
    print(json.dumps({"config": name, "N": N, "K": K, "prec": prec, "kernel": s.kernel, **out}), flush=True)
