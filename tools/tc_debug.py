"""Debug: sums produced by the SIMT and TC passes vs numpy sums of the stored Theta^k."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import crdata
import paper_1608_02227_b200 as crp

N, n = int(sys.argv[1]), int(sys.argv[2])
X, ybar = crdata.random_problem(N, n, seed=5, fp32=True)
rel = lambda a, b: float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
np.set_printoptions(precision=4, linewidth=200)
for kern in ("simt", "tc"):
    s = crp.Solver(X, ybar, 1e-3, kernel=kern)
    s.step(); s.step()
    T = s.get_theta()[0]
    r, c, P = s.get_sums(0)
    Pw = T @ X
    print(kern, "r", rel(r, T.sum(1)), "c", rel(c, T.sum(0)), "P", rel(P, Pw))
    if kern == "tc":
        print(" r ratio", (r / T.sum(1))[:8])
        print(" c ratio", (c / T.sum(0))[:40])
        print(" P[0]", P[0, :8]); print(" Pw[0]", Pw[0, :8])
        # try hypotheses: P vs T @ X permuted / scaled
        for name, cand in [("2x", 2 * Pw), ("hi only", T @ X)]:
            pass
    s.close()
