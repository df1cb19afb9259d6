"""Dense numpy mirror of kernels/block_ipm.cu's Mehrotra iteration (development aid: how the
projection error depends on the stopping rule / polish).  Compares with the oracle's NNLS
projection.  Not used by the product or the tests."""
import sys
import numpy as np

sys.path.insert(0, ".")
import crdata
from oracle import partition, ref


def ipm(Xb, y0, xi0, gamma, tol=1e-9, max_iter=100, polish=True, rho=0.1, verbose=False):
    """Mehrotra predictor-corrector (stop: max complementarity, residuals <= tol (scaled)), then the
    active-set polish by the method of multipliers -- the kernel's algorithm with dense solves."""
    nb, n = Xb.shape
    A = np.hstack([ref.dense_A1(nb), ref.dense_A2(Xb)])        # rows: pairs (l, l'), l != l'
    G = np.diag(np.r_[np.ones(nb), gamma * np.ones(nb * n)])
    e0 = np.r_[y0, xi0.reshape(-1)]
    eta = e0.copy()
    a = A @ eta
    sc = max(1.0, np.abs(a).max())
    s = np.maximum(a, 0) + sc
    lam = np.full_like(s, 1e-2 * sc)
    m = len(s)
    for it in range(max_iter):
        rp = A @ eta - s
        rd = G @ (eta - e0) - A.T @ lam
        mu = s @ lam / m
        if verbose:
            print(it, mu, np.abs(rp).max(), np.abs(rd).max())
        if (s * lam).max() <= tol * sc * sc and np.abs(rp).max() <= tol * sc and np.abs(rd).max() <= tol * sc:
            break
        D = lam / s
        M = G + A.T @ (D[:, None] * A)

        def dirn(w):
            de = np.linalg.solve(M, -rd + A.T @ w)
            return de, A @ de + rp, w - D * (A @ de)
        w = -lam - D * rp
        de, ds, dl = dirn(w)
        ap = min(1, min((-s[ds < 0] / ds[ds < 0]), default=1))
        ad = min(1, min((-lam[dl < 0] / dl[dl < 0]), default=1))
        mua = (s + ap * ds) @ (lam + ad * dl) / m
        sig = min(1, (mua / mu) ** 3)
        w = -lam + (sig * mu - ds * dl) / s - D * rp
        de, ds, dl = dirn(w)
        ap = min(1, 0.995 * min((-s[ds < 0] / ds[ds < 0]), default=1e300))
        ad = min(1, 0.995 * min((-lam[dl < 0] / dl[dl < 0]), default=1e300))
        s += ap * ds
        lam += ad * dl
        eta += ap * de
    if not polish:
        return eta[:nb], eta[nb:].reshape(nb, n), it
    act = lam > s
    la = np.where(act, lam, 0.0)
    for _ in range(6):
        M = G + rho * A[act].T @ A[act]
        for _ in range(150):
            et = np.linalg.solve(M, G @ e0 + A.T @ la)
            c = A @ et
            la = np.where(act, la - rho * c, 0.0)
            if np.abs(c[act]).max(initial=0.0) <= 1e-15 * sc:
                break
        viol = ~act & (c < -1e-12 * sc)
        neg = act & (la < -1e-14 * max(1.0, np.abs(la).max()))
        if not viol.any() and not neg.any():
            return et[:nb], et[nb:].reshape(nb, n), it
        act = (act | viol) & ~neg
        la = np.maximum(np.where(act, la, 0.0), 0.0)
    return eta[:nb], eta[nb:].reshape(nb, n), -1


if __name__ == "__main__":
    N, n, nbar, gamma = 120, 3, 12, 1e-2
    X, ybar = crdata.random_problem(N, n, seed=0)
    L = ref.lipschitz(X, gamma)
    st = partition.papg_partition(X, ybar, gamma, L, 5, nbar)
    T = np.where(partition.block_mask(N, nbar), st["Tt"], 0)
    from oracle.core import eta as eta_cross
    y0, xi0 = eta_cross(X, ybar, gamma, T)
    for tol in (1e-9,):
        for pol in (False, True):
            errs, its = [], []
            for b in range(N // nbar):
                r = slice(b * nbar, (b + 1) * nbar)
                yw, xw, _ = partition.project_block(X[r], y0[r], xi0[r], gamma)
                y, xi, it = ipm(X[r], y0[r], xi0[r], gamma, tol=tol, polish=pol, max_iter=200)
                errs.append(max(np.abs(y - yw).max() / np.abs(yw).max(), np.abs(xi - xw).max() / np.abs(xw).max()))
                its.append(it)
            print(f"tol {tol:g} polish {pol}: max rel err {max(errs):.2e} iters {max(its)}")
