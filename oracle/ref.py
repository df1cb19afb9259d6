"""Dense / library-routine references -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Every function cites the PAPER.md passage it writes out.  Dense matrices are
only built for tiny N (N <= ~60).
"""
from __future__ import annotations

import numpy as np
import scipy.optimize
import scipy.sparse.linalg as sla


# ---------------------------------------------------------------------------
# Def. A1A2: T_l = [e_1 ... e_{l-1}  -1  e_l ... e_{N-1}] in R^{(N-1) x N},
# A1 = [T_1; ...; T_N],  A2 = diag(X_1, ..., X_N),  X_l = -T_l Xbar.
# Rows in lexicographic order of (l1, l2), l1 != l2.
# ---------------------------------------------------------------------------
def T_matrix(N: int, l: int) -> np.ndarray:
    """T_l for 0-based l (the paper's l+1)."""
    T = np.zeros((N - 1, N))
    for c in range(N):
        if c < l:
            T[c, c] = 1.0          # e_{c+1} occupies column c
        elif c == l:
            T[:, c] = -1.0         # the -1 column
        else:
            T[c - 1, c] = 1.0      # e_c after the -1 column
    return T


def dense_A1(N: int) -> np.ndarray:
    return np.vstack([T_matrix(N, l) for l in range(N)])


def dense_A2(X: np.ndarray) -> np.ndarray:
    N, n = X.shape
    A2 = np.zeros((N * (N - 1), N * n))
    for l in range(N):
        A2[l * (N - 1):(l + 1) * (N - 1), l * n:(l + 1) * n] = -T_matrix(N, l) @ X
    return A2


def dense_C(X: np.ndarray) -> np.ndarray:
    """C = [A3 A4] = [A1 A2] when every pair is dualized (Def. C, P:345-350 with K = N)."""
    return np.hstack([dense_A1(X.shape[0]), dense_A2(X)])


def pair_index(i: int, j: int, N: int) -> int:
    """Row of pair (l1, l2) = (i, j), i != j, in the lexicographic order of P:101-102."""
    return i * (N - 1) + j - (1 if j > i else 0)


def theta_vec(Theta: np.ndarray) -> np.ndarray:
    """Dense N x N (zero diagonal) -> packed theta in R^{N(N-1)} (lexicographic)."""
    N = Theta.shape[0]
    return Theta[~np.eye(N, dtype=bool)].copy()


def theta_mat(theta: np.ndarray, N: int) -> np.ndarray:
    T = np.zeros((N, N))
    T[~np.eye(N, dtype=bool)] = theta
    return T


# ---------------------------------------------------------------------------
# Dual function, dense (Eq. (g_gamma), Eq. (dual gradient) P:367-371)
# ---------------------------------------------------------------------------
def eta_dense(theta: np.ndarray, X: np.ndarray, ybar: np.ndarray, gamma: float):
    """argmin_eta 1/2||y-ybar||^2 + gamma/2||xi||^2 - <theta, C eta> (Step 1; Q = R^{N(n+1)}).

    Stationarity: y - ybar - A1^T theta = 0, gamma xi - A2^T theta = 0.
    """
    N, n = X.shape
    y = ybar + dense_A1(N).T @ theta
    xi = (dense_A2(X).T @ theta) / gamma
    return y, xi.reshape(N, n)


def lagrangian_dense(y, xi, theta, X, ybar, gamma):
    """L_gamma(y, xi, theta), Eq. (lagrangian) P:159-161 with every pair dualized."""
    Ceta = dense_A1(len(y)) @ y + dense_A2(X) @ xi.reshape(-1)
    return 0.5 * np.sum((y - ybar) ** 2) + 0.5 * gamma * np.sum(xi ** 2) - theta @ Ceta


def dual_value_dense(theta, X, ybar, gamma):
    """g_gamma(theta) = min_eta L_gamma (Eq. (g_gamma)), at the closed-form minimizer."""
    y, xi = eta_dense(theta, X, ybar, gamma)
    return lagrangian_dense(y, xi, theta, X, ybar, gamma)


def dual_grad_dense(theta, X, ybar, gamma):
    """grad g_gamma(theta) = -C eta(theta) (Eq. (dual gradient) P:370)."""
    y, xi = eta_dense(theta, X, ybar, gamma)
    return -(dense_A1(len(y)) @ y + dense_A2(X) @ xi.reshape(-1))


# ---------------------------------------------------------------------------
# Exact regularized optimum (Eq. (regularize), dual P:168-177).
# max_{theta>=0} g(theta)  <=>  min_{theta>=0} 1/2 || [A1^T; A2^T/sqrt(gamma)] theta - [-ybar; 0] ||^2
# (expand g at its minimizer: g = -1/2||A1^T th||^2 - 1/(2 gamma)||A2^T th||^2 - ybar^T A1^T th).
# Solved by Lawson-Hanson NNLS (scipy.optimize.nnls); eta* = eta(theta*) (strong duality).
# ---------------------------------------------------------------------------
def regularized_optimum(X, ybar, gamma, maxiter=None):
    N, n = X.shape
    A1, A2 = dense_A1(N), dense_A2(X)
    M = np.vstack([A1.T, A2.T / np.sqrt(gamma)])
    b = np.concatenate([-ybar, np.zeros(N * n)])
    theta, _ = scipy.optimize.nnls(M, b, maxiter=maxiter if maxiter else 50 * M.shape[1])
    y, xi = eta_dense(theta, X, ybar, gamma)
    p = 0.5 * np.sum((y - ybar) ** 2) + 0.5 * gamma * np.sum(xi ** 2)
    return dict(theta=theta, y=y, xi=xi, p=p)


# ---------------------------------------------------------------------------
# Univariate convex LS fit (pin for Lemma 1): sorted x, slopes
# nondecreasing  <=>  D y >= 0 with D the scaled second-difference operator.
# Dual: y = ybar + D^T lam, lam = argmin_{lam>=0} 1/2||D^T lam + ybar||^2 (NNLS).
# ---------------------------------------------------------------------------
def convex_fit_1d(x, ybar):
    x = np.asarray(x, dtype=np.float64)
    order = np.argsort(x)
    xs, ys = x[order], np.asarray(ybar, dtype=np.float64)[order]
    N = len(xs)
    D = np.zeros((N - 2, N))
    for k in range(1, N - 1):
        h0, h1 = xs[k] - xs[k - 1], xs[k + 1] - xs[k]
        D[k - 1, k - 1] = 1.0 / h0
        D[k - 1, k] = -1.0 / h0 - 1.0 / h1
        D[k - 1, k + 1] = 1.0 / h1
    lam, _ = scipy.optimize.nnls(D.T, -ys, maxiter=100 * N)
    yfit = np.empty(N)
    yfit[order] = ys + D.T @ lam
    return yfit


# ---------------------------------------------------------------------------
# L_gamma = sigma_max(C)^2 / gamma   (Eq. (lischitz)).
# sigma_max(C)^2 = lambda_max(C^T C), computed by ARPACK Lanczos (scipy eigsh)
# on a matrix-free C^T C.  Two forms of the product:
#   "definition": z = C v pair by pair (row chunks, O(N^2 n)), then C^T z
#   "structured": O(N n^2) rearrangement of the same sums (derived;
#                 pinned against "definition" in tests/test_oracle_pins.py)
# ---------------------------------------------------------------------------
def CtC_definition(X, v, chunk=1024):
    N, n = X.shape
    y, xi = v[:N], v[N:].reshape(N, n)
    a = np.einsum("ij,ij->i", xi, X)
    colsum = np.zeros(N)
    out_y = np.zeros(N)
    out_xi = np.zeros((N, n))
    for i0 in range(0, N, chunk):
        i1 = min(N, i0 + chunk)
        # z_ij = y_j - y_i + xi_i^T (x_i - x_j)   (pair constraint)
        Z = y[None, :] - y[i0:i1, None] + a[i0:i1, None] - xi[i0:i1] @ X.T
        Z[np.arange(i1 - i0), np.arange(i0, i1)] = 0.0
        rs = Z.sum(axis=1)
        colsum += Z.sum(axis=0)
        out_y[i0:i1] -= rs                                 # A1^T z: - row sums
        out_xi[i0:i1] = rs[:, None] * X[i0:i1] - Z @ X     # A2^T z: sum_j z_ij (x_i - x_j)
    out_y += colsum                                        # A1^T z: + column sums
    return np.concatenate([out_y, out_xi.reshape(-1)])


def CtC_structured(X, v):
    N, n = X.shape
    y, xi = v[:N], v[N:].reshape(N, n)
    a = np.einsum("ij,ij->i", xi, X)
    s = X.sum(axis=0)
    Y, Sa = y.sum(), a.sum()
    Sxi = xi.sum(axis=0)
    w = X.T @ y
    S2 = X.T @ X
    xs = xi @ s
    rho = Y - N * y + N * a - xs                           # row sums of z
    out_y = 2 * N * y - 2 * Y + Sa - X @ Sxi - N * a + xs
    out_xi = X * rho[:, None] - w[None, :] + (y - a)[:, None] * s[None, :] + xi @ S2
    return np.concatenate([out_y, out_xi.reshape(-1)])


def sigma_max_sq(X, form="auto", tol=1e-13):
    N, n = X.shape
    if form == "auto":
        form = "definition" if N <= 4096 else "structured"
    mv = (lambda v: CtC_definition(X, v)) if form == "definition" else (lambda v: CtC_structured(X, v))
    dim = N * (n + 1)
    if dim <= 40:
        M = np.column_stack([mv(e) for e in np.eye(dim)])
        return float(np.linalg.eigvalsh(0.5 * (M + M.T))[-1])
    op = sla.LinearOperator((dim, dim), matvec=mv, dtype=np.float64)
    v0 = np.random.default_rng(12345).standard_normal(dim)
    w = sla.eigsh(op, k=1, which="LA", tol=tol, v0=v0, return_eigenvectors=False, ncv=min(dim - 1, 40))
    return float(w[0])


def lipschitz(X, gamma, form="auto"):
    """L_gamma = sigma_max^2(C) / gamma (Eq. (lischitz))."""
    return sigma_max_sq(X, form) / gamma


# ---------------------------------------------------------------------------
# The fitted estimator (Eq. (original) and the piecewise-linear interpolant it
# certifies): a feasible (y, xi) defines the max-affine function
#     f_hat(z) = max_i  y_i + xi_i^T (z - x_i),
# which interpolates y at the data points when every pair constraint holds.
# ---------------------------------------------------------------------------
def predict(X, y, xi, Z):
    """f_hat at the rows of Z (M x n), written out as the definition (fp64)."""
    X, y, xi, Z = (np.asarray(a, dtype=np.float64) for a in (X, y, xi, Z))
    out = np.empty(Z.shape[0])
    for m in range(Z.shape[0]):
        out[m] = np.max(y + np.einsum("ij,ij->i", xi, Z[m][None, :] - X))
    return out
