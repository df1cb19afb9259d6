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
    out = []
    # exact fp64 run (one state, advanced in place)
    EP, EQ = np.zeros((N, N)), np.zeros((N, N))
    et = 1.0
    # fp32-storage run: Theta^k rounded to fp32 once per iteration, theta~^{k+1} re-formed from the
    # stored iterates (Step 4) as the GPU does
    P, Q = np.zeros((N, N)), np.zeros((N, N))
    t = 1.0
    done = 0
    for K in ks:
        et = oracle.papg(X, ybar, cfg.gamma, L, K - done, Tprev=EP, Tt=EQ, t=et, inplace=True)["t"]
        for _ in range(K - done):
            prev = P.copy()
            tn = oracle.papg(X, ybar, cfg.gamma, L, 1, Tprev=P, Tt=Q, t=t, inplace=True)["t"]
            P[...] = P.astype(np.float32)                          # fp32 storage of Theta^k
            Q[...] = oracle.extrapolate(P, prev, t, tn)
            t = tn
        done = K
        ya, xa = oracle.eta(X, ybar, cfg.gamma, EP)
        sa = oracle.stats(X, ybar, cfg.gamma, EP, ya, xa)
        yb, xb = oracle.eta(X, ybar, cfg.gamma, P)
        sb = oracle.stats(X, ybar, cfg.gamma, P, yb, xb)
        rec = {"config": name, "N": N, "K": K,
               **{k: abs(sb[k] - sa[k]) / max(abs(sa[k]), 1e-300) for k in sa}}
        out.append(rec)
        print(json.dumps(rec), flush=True)
    return out


GOLDEN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "golden",
                      "fp32_storage_floor.json")


def write_golden(recs):
    """Merge records into tests/golden/fp32_storage_floor.json (the K-iteration parity tests read
    their max-violation tolerance from it)."""
    doc = {"_source": "Written by tests/numerics/fp32_storage_floor.py (oracle/ only): relative change of "
                      "eta(Theta^K)'s diagnostics (Theorem 1 P:241-247, P:1104-1106) when Theta^k is rounded to "
                      "fp32 once per iteration of Fig. 2 (P:377-397), every other operation fp64.  DESIGN.md "
                      "§Numerics.", "records": []}
    if os.path.exists(GOLDEN):
        doc = json.load(open(GOLDEN))
    keep = [r for r in doc["records"] if not any((r["config"], r["N"], r["K"]) == (q["config"], q["N"], q["K"])
                                                 for q in recs)]
    doc["records"] = sorted(keep + recs, key=lambda r: (r["config"], r["N"], r["K"]))
    with open(GOLDEN, "w") as f:
        json.dump(doc, f, indent=1)


if __name__ == "__main__":
    nm = sys.argv[1] if len(sys.argv) > 1 else "C2"
    kk = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "500,1000,2000").split(",")]
    recs = run_floor(nm, kk, N=int(os.environ["FLOOR_N"]) if "FLOOR_N" in os.environ else None)
    if "--write" in sys.argv:
        write_golden(recs)
