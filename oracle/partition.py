"""P-APG with a general partition K < N (Section 2; Fig. 2) -- TEST
INFRASTRUCTURE ONLY (see oracle/__init__.py).

Assumption 1: N = K Nbar, blocks C_i = {(i-1) Nbar + 1, ..., i Nbar} (0-based here:
rows [i Nbar, (i+1) Nbar)).  Only the cross-block pair constraints are dualized (theta_ij for
l1, l2 in different blocks, Eq. (lagrangian)); the intra-block constraints stay in the
subproblems (Eq. (subgradient_split)).  Step 1 is therefore, per block i,

    min  1/2 ||y_i - ybar_i||^2 + gamma/2 ||xi_i||^2 - <theta, A1^{.i} y + A2^{.i} xi>   s.t.  Abar^ii eta_i >= 0

= the G-norm projection (G = diag(I, gamma I)) of the unconstrained minimizer eta0 = (ybar + A1^T theta,
A2^T theta / gamma) onto Q_i.  This oracle solves each projection EXACTLY through its dual, a
nonnegative least-squares problem (Lawson-Hanson, scipy.optimize.nnls):
    lambda = argmin_{lambda >= 0} 1/2 || [A1b^T ; A2b^T / sqrt(gamma)] lambda + [y0_b ; sqrt(gamma) xi0_b] ||^2,
    y_b = y0_b + A1b^T lambda,   xi_b = xi0_b + A2b^T lambda / gamma
(A1b, A2b: Def. A1A2 P:103-128 on the block's points).  Steps 2-4 as in Fig. 2 on the cross-block
entries; intra-block entries of Theta are identically 0.
"""
from __future__ import annotations

import numpy as np
import scipy.optimize

from . import ref
from .core import eta as _eta_cross, momentum_next


def _check(N, nbar):
    if nbar < 1 or N % nbar:
        raise ValueError("Assumption 1 (P:141): N = K * Nbar")


def block_mask(N: int, nbar: int) -> np.ndarray:
    """True on the cross-block pairs (the dualized constraints), False on intra-block ones."""
    b = np.arange(N) // nbar
    return b[:, None] != b[None, :]


def project_block(Xb, y0, xi0, gamma):
    """G-norm projection of (y0, xi0) onto Q_i = {Abar^ii eta >= 0} for one block (exact, NNLS dual)."""
    m = Xb.shape[0]
    A1, A2 = ref.dense_A1(m), ref.dense_A2(Xb)
    M = np.vstack([A1.T, A2.T / np.sqrt(gamma)])
    t = -np.concatenate([y0, np.sqrt(gamma) * xi0.reshape(-1)])
    lam, _ = scipy.optimize.nnls(M, t, maxiter=100 * M.shape[1])
    y = y0 + A1.T @ lam
    xi = xi0.reshape(-1) + (A2.T @ lam) / gamma
    return y, xi.reshape(xi0.shape), lam


def step1(X, ybar, gamma, Tt, nbar):
    """Step 1 for the partition: per-block projections of the closed-form point."""
    N = X.shape[0]
    _check(N, nbar)
    T = np.where(block_mask(N, nbar), Tt, 0.0)
    y0, xi0 = _eta_cross(X, ybar, gamma, T)          # ybar + A1^T theta, A2^T theta / gamma
    if nbar == 1:
        return y0, xi0
    y, xi = y0.copy(), xi0.copy()
    for b in range(N // nbar):
        r = slice(b * nbar, (b + 1) * nbar)
        y[r], xi[r], _ = project_block(X[r], y0[r], xi0[r], gamma)
    return y, xi


def papg_partition(X, ybar, gamma, L, K, nbar, Tprev=None, Tt=None, t=1.0):
    """K iterations of Fig. 2 with blocks of nbar points; state as oracle.papg."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    N = X.shape[0]
    _check(N, nbar)
    mask = block_mask(N, nbar)
    Tprev = np.zeros((N, N)) if Tprev is None else np.array(Tprev, dtype=np.float64)
    Tt = Tprev.copy() if Tt is None else np.array(Tt, dtype=np.float64)
    y = xi = None
    for _ in range(K):
        y, xi = step1(X, ybar, gamma, Tt, nbar)                       # Step 1
        R = y[None, :] - y[:, None] + np.einsum("id,id->i", xi, X)[:, None] - xi @ X.T   # (C eta)_ij
        Tn = np.where(mask, np.maximum(Tt - R / L, 0.0), 0.0)          # Step 2, cross-block only
        tn = momentum_next(t)                                          # Step 3
        Tt = Tn + ((t - 1.0) / tn) * (Tn - Tprev)                      # Step 4
        Tprev, t = Tn, tn
    return dict(Tprev=Tprev, Tt=Tt, t=t, y=y, xi=xi)


def eta_partition(X, ybar, gamma, T, nbar):
    """eta(Theta) for the partition (Theorem 1's estimator): Step 1 at Theta."""
    return step1(np.ascontiguousarray(X, dtype=np.float64), ybar, gamma, T, nbar)
