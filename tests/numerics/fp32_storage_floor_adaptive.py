"""fp32-storage numerics floor of the ADAPTIVE P-APG run.

Runs the oracle's adaptive iteration with every operation in fp64 except that Theta^k is
rounded to fp32 once per iteration (the storage precision of the fp32 configs), and reports
how far Theta^K and the diagnostics of eta(Theta^K) move from the pure fp64 oracle run, and
whether the accept/reject decisions stay identical.  Uses only oracle/ and crdata.

    python tests/numerics/fp32_storage_floor_adaptive.py 300,5,25 1000,20,25
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

import crdata  # noqa: E402
import oracle  # noqa: E402
from oracle import ref  # noqa: E402


def floor(N, n, K, gamma=1e-3, seed=None):
    X, ybar = crdata.random_problem(N, n, seed=N + n if seed is None else seed, fp32=True)
    L = ref.lipschitz(X, gamma)
    r32 = lambda a: a.astype(np.float32).astype(np.float64)
    ex = oracle.papg_adaptive(X, ybar, gamma, L, K)
    st = dict(Tprev=np.zeros((N, N)), Tt=np.zeros((N, N)), t=1.0, s=L)
    trials = []
    for _ in range(K):
        o = oracle.papg_adaptive(X, ybar, gamma, st["s"], 1, Tprev=st["Tprev"], Tt=st["Tt"], t=st["t"])
        trials.append(int(o["trials"][0]))
        Tk = r32(o["Tprev"])
        st = dict(Tprev=Tk, Tt=oracle.extrapolate(Tk, st["Tprev"], st["t"], o["t"]), t=o["t"], s=o["s"])
    sa = oracle.stats(X, ybar, gamma, st["Tprev"], *oracle.eta(X, ybar, gamma, st["Tprev"]))
    sb = oracle.stats(X, ybar, gamma, ex["Tprev"], *oracle.eta(X, ybar, gamma, ex["Tprev"]))
    return dict(theta=float(np.linalg.norm(st["Tprev"] - ex["Tprev"]) / np.linalg.norm(ex["Tprev"])),
                objective=abs(sa["r_gamma"] - sb["r_gamma"]) / abs(sb["r_gamma"]),
                max_violation=abs(sa["max_violation"] - sb["max_violation"]) / abs(sb["max_violation"]),
                same_decisions=trials == [int(v) for v in ex["trials"]])


if __name__ == "__main__":
    for arg in sys.argv[1:] or ["300,5,25"]:
        N, n, K = (int(v) for v in arg.split(","))
        print(arg, floor(N, n, K))
