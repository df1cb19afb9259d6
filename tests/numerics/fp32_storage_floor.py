"""Numerics floor of fp32 Theta storage.

Runs the P-APG iteration of Fig. 2 with every operation in fp64 EXCEPT that Theta^k is
rounded to fp32 once per iteration (the storage precision BASELINE.json fixes for C2-C5),
and reports how far eta(Theta^K)'s diagnostics move from the pure fp64 oracle.  Any fp32-
storage implementation inherits at least this drift.  Uses only oracle/ (fp64 reference) and
numpy; the CUDA path is not involved.

    python tests/numerics/fp32_storage_floor.py C2 500,1000,2000
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

import crdata  # noqa: E402
import oracle  # noqa: E402
from oracle import ref  # noqa: E402


def run_floor(name, ks, N=None):
    cfg = crdata.CONFIGS[name]
    X, ybar = crdata.make_problem(cfg, N=N)
    N = X.shape[0]
    L = ref.lipschitz(X, cfg.gamma)
    r32 = lambda a: a.astype(np.float32).astype(np.float64)
    out = []
    ex = oracle.papg(X, ybar, cfg.gamma, L, 0)
    st = dict(Tprev=np.zeros((N, N)), Tt=np.zeros((N, N)), t=1.0)
    done = 0
    for K in ks:
        ex = oracle.papg(X, ybar, cfg.gamma, L, K - done, Tprev=ex["Tprev"], Tt=ex["Tt"], t=ex["t"])
        for _ in range(K - done):
            prev = st["Tprev"]
            o = oracle.papg(X, ybar, cfg.gamma, L, 1, Tprev=st["Tprev"], Tt=st["Tt"], t=st["t"])
            Tk = r32(o["Tprev"])                                   # fp32 storage of Theta^k
            # theta~^{k+1} re-formed from the stored iterates (Step 4), as the GPU does
            tk = st["t"]
            st = dict(Tprev=Tk, Tt=oracle.extrapolate(Tk, prev, tk, o["t"]), t=o["t"])
        done = K
        ya, xa = oracle.eta(X, ybar, cfg.gamma, ex["Tprev"])
        sa = oracle.stats(X, ybar, cfg.gamma, ex["Tprev"], ya, xa)
        yb, xb = oracle.eta(X, ybar, cfg.gamma, st["Tprev"])
        sb = oracle.stats(X, ybar, cfg.gamma, st["Tprev"], yb, xb)
        rec = {"config": name, "N": N, "K": K,
               **{k: abs(sb[k] - sa[k]) / max(abs(sa[k]), 1e-300) for k in sa}}
        out.append(rec)
        print(json.dumps(rec), flush=True)
    return out


if __name__ == "__main__":
    nm = sys.argv[1] if len(sys.argv) > 1 else "C2"
    kk = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "500,1000,2000").split(",")]
    run_floor(nm, kk, N=int(os.environ["FLOOR_N"]) if "FLOOR_N" in os.environ else None)
