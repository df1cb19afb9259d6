import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, crdata
import paper_1608_02227_b200 as crp
for cfg_name, K in (("C4", 1000), ("C3", 2000), ("C5", 200)):
    c = crdata.CONFIGS[cfg_name]
    X, ybar = crdata.make_problem(c)
    s = crp.Solver(X, ybar, c.gamma, prec=c.prec)
    res = []
    for done in (K // 10, K // 2, K):
        s.solve(done - sum(r[0] for r in res[-1:]) if res else done)
        rows = np.random.default_rng(0).choice(c.N // 128, size=min(8, c.N // 128), replace=False)
        nz = 0; zt = 0; tot = 0
        for rb in rows:
            T = s.get_theta_rows(0, int(rb) * 128, 128)
            nz += np.count_nonzero(T)
            tiles = T[:, : (c.N // 32) * 32].reshape(128, -1, 32)
            z = np.all(tiles == 0, axis=(0, 2))
            zt += z.sum(); tot += z.size
        res.append((done, nz / (len(rows) * 128 * c.N), zt / tot))
        print(cfg_name, "iter", done, "nonzero frac %.4f" % res[-1][1], "all-zero 128x32 tiles %.4f" % res[-1][2], flush=True)
    s.close()
