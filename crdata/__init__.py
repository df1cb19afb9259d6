"""Seeded synthetic inputs shared by the oracle, the tests and the bench.

This module is the ONLY code shared between ``oracle/`` and the CUDA path.
It holds none of the method's arithmetic: it draws observations
{(x_l, ybar_l)} (PAPER.md Eq. (data)) and, for tests, random
nonnegative multiplier states.  Everything the P-APG iteration computes lives
in ``oracle/`` (reference) and ``paper_1608_02227_b200/`` (product).

Configs C1-C5 follow BASELINE.json ``configs`` and SURVEY.md §8(d).  Where
BASELINE.json is silent (gamma for C2-C5, seeds, the LSE piece law of C4) the
readings of DESIGN.md §"Readings" apply: gamma = 1e-3, numpy PCG64
``default_rng(seed)`` with seed 0, draw order X -> f0 parameters -> noise.
fp32 configs round X and ybar to float32 (then promote to float64) so both
sides see the identical problem.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

__all__ = ["Config", "CONFIGS", "make_problem", "random_problem", "random_theta", "paper_problem"]


@dataclass(frozen=True)
class Config:
    name: str
    N: int
    n: int
    prec: str          # "fp64" | "fp32": storage / elementwise precision of the GPU path
    x_law: str         # "uniform" (U[-1,1]^n) | "normal" (N(0, I_n))
    f0: str            # "sqnorm" | "maxaffine" | "lse"
    f0_scale: float    # f0 = ||x||^2 * f0_scale for "sqnorm"
    pieces: int        # affine pieces for maxaffine / lse
    noise_sd: float
    gamma: float
    iters: int
    gpus: tuple = field(default=(1,))


CONFIGS = {
    "C1": Config("C1", 50, 2, "fp64", "uniform", "sqnorm", 1.0, 0, 0.1, 1e-3, 500),
    "C2": Config("C2", 1000, 10, "fp32", "normal", "maxaffine", 0.0, 8, 0.3, 1e-3, 2000),
    "C3": Config("C3", 4000, 20, "fp32", "uniform", "sqnorm", 1.0 / 20, 0, 0.1, 1e-3, 2000, (1, 2, 4, 8)),
    "C4": Config("C4", 16384, 40, "fp32", "normal", "lse", 0.0, 16, 0.2, 1e-3, 1000, (1, 2, 4, 8)),
    "C5": Config("C5", 65536, 80, "fp32", "uniform", "sqnorm", 1.0 / 80, 0, 0.1, 1e-3, 200, (1, 2, 4, 8)),
}


def _draw_x(rng, law, N, n):
    if law == "uniform":
        return rng.uniform(-1.0, 1.0, size=(N, n))
    if law == "normal":
        return rng.standard_normal(size=(N, n))
    raise ValueError(law)


def _f0(rng, cfg, X):
    """Ground-truth convex function values (data generation only)."""
    if cfg.f0 == "sqnorm":
        return cfg.f0_scale * np.einsum("ij,ij->i", X, X)
    A = rng.standard_normal(size=(cfg.pieces, X.shape[1]))   # slopes  N(0, I)
    b = rng.standard_normal(size=cfg.pieces)                 # offsets N(0, 1)
    Z = X @ A.T + b
    if cfg.f0 == "maxaffine":
        return Z.max(axis=1)
    if cfg.f0 == "lse":
        m = Z.max(axis=1, keepdims=True)
        return (m + np.log(np.exp(Z - m).sum(axis=1, keepdims=True)))[:, 0]
    raise ValueError(cfg.f0)


def make_problem(cfg: Config | str, seed: int = 0, N: int | None = None):
    """Return (X [N,n] float64 C-contiguous, ybar [N] float64) for a config.

    ``N`` overrides the config size (same laws) for reduced-size parity cases.
    fp32 configs return float32-representable values promoted to float64.
    """
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    N = cfg.N if N is None else int(N)
    rng = np.random.default_rng(seed)
    X = _draw_x(rng, cfg.x_law, N, cfg.n)
    f = _f0(rng, cfg, X)
    ybar = f + cfg.noise_sd * rng.standard_normal(size=N)
    if cfg.prec == "fp32":
        X = X.astype(np.float32).astype(np.float64)
        ybar = ybar.astype(np.float32).astype(np.float64)
    return np.ascontiguousarray(X), np.ascontiguousarray(ybar)


def random_problem(N: int, n: int, seed: int = 0, law: str = "normal", noise_sd: float = 0.3,
                   fp32: bool = False):
    """Small random instance: x ~ law, ybar = ||x||^2 + noise (convex truth + noise)."""
    rng = np.random.default_rng(seed)
    X = _draw_x(rng, law, N, n)
    ybar = np.einsum("ij,ij->i", X, X) + noise_sd * rng.standard_normal(size=N)
    if fp32:
        X = X.astype(np.float32).astype(np.float64)
        ybar = ybar.astype(np.float32).astype(np.float64)
    return np.ascontiguousarray(X), np.ascontiguousarray(ybar)


def random_theta(N: int, seed: int = 0, scale: float = 1.0, density: float = 0.5, fp32: bool = False):
    """Random nonnegative N x N multiplier matrix with zero diagonal (a valid dual point)."""
    rng = np.random.default_rng(seed)
    T = rng.exponential(scale, size=(N, N)) * (rng.uniform(size=(N, N)) < density)
    np.fill_diagonal(T, 0.0)
    if fp32:
        T = T.astype(np.float32).astype(np.float64)
    return np.ascontiguousarray(T)


def paper_problem(N: int, n: int, f0: str = "quad", seed: int = 0):
    """The synthetic workload of the paper's Section 4, for context runs only:
    f0 = 1/2 x^T Q x ("quad": Q = Lambda^T Lambda, Lambda iid N(0,1), singular values mapped
    affinely onto [s_max/15, s_max] so cond(Q) = 15 -- the paper does not say how it transforms
    them) or f0 = exp(p^T x) ("exp": p ~ U[0, 0.2]^n); x iid N(0, 4), eps iid N(0, 100),
    ybar = f0(x) + eps, then 30% of the points (chosen at random) get ybar <- 1.3 ybar.
    Draw order: X, f0 parameters, noise, the 30% subset.  Returns (X, ybar) in float64."""
    rng = np.random.default_rng(seed)
    X = 2.0 * rng.standard_normal(size=(N, n))
    if f0 == "quad":
        Lam = rng.standard_normal(size=(n, n))
        U, sv, Vt = np.linalg.svd(Lam.T @ Lam)
        smax, smin = sv.max(), sv.min()
        lo = smax / 15.0
        sv2 = lo + (sv - smin) * (smax - lo) / max(smax - smin, 1e-300)
        Q = (U * sv2) @ Vt
        Q = 0.5 * (Q + Q.T)
        f = 0.5 * np.einsum("ij,jk,ik->i", X, Q, X)
    elif f0 == "exp":
        pv = rng.uniform(0.0, 0.2, size=n)
        f = np.exp(X @ pv)
    else:
        raise ValueError(f0)
    ybar = f + 10.0 * rng.standard_normal(size=N)
    moved = rng.choice(N, size=int(round(0.3 * N)), replace=False)
    ybar[moved] *= 1.3
    return np.ascontiguousarray(X), np.ascontiguousarray(ybar)
