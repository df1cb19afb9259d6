"""ctypes wrapper for oracle/papg_oracle.c -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py)."""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "papg_oracle.c")
_SO = os.path.join(_HERE, "libpapg_oracle.so")
_lib = None

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")


def build_oracle(force: bool = False) -> str:
    """Compile the fp64 oracle: gcc -O2 -fopenmp (no -ffast-math, no intrinsics)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               _SRC, "-o", _SO, "-lm"])
    return _SO


def lib():
    global _lib
    if _lib is None:
        build_oracle()
        L = C.CDLL(_SO)
        i64, i32, d = C.c_int64, C.c_int, C.c_double
        dpn = C.c_void_p  # nullable double*
        L.oracle_papg.argtypes = [i64, i32, _dp, _dp, d, d, i64, _dp, _dp, C.POINTER(d), dpn, dpn, i32]
        L.oracle_eta.argtypes = [i64, i32, _dp, _dp, d, _dp, _dp, _dp, i32]
        L.oracle_stats.argtypes = [i64, i32, _dp, _dp, d, dpn, _dp, _dp, _dp, i32]
        L.oracle_project_rows.argtypes = [i64, i32, _dp, _dp, _dp, d, _ip, i64, _dp, _dp, i32]
        L.oracle_papg_adaptive.argtypes = [i64, i32, _dp, _dp, d, d, i64, _dp, _dp, C.POINTER(d), C.POINTER(d),
                                           _ip, _dp, dpn, dpn, i32, i32, i32]
        for f in (L.oracle_papg, L.oracle_eta, L.oracle_stats, L.oracle_project_rows, L.oracle_papg_adaptive):
            f.restype = C.c_int
        L.oracle_max_threads.restype = C.c_int
        _lib = L
    return _lib


def max_threads() -> int:
    return int(lib().oracle_max_threads())


def _c64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def momentum_next(t: float) -> float:
    """Step 3 of Fig. 2: t_{k+1} = (1 + sqrt(1 + 4 t_k^2)) / 2."""
    return (1.0 + math.sqrt(1.0 + 4.0 * t * t)) / 2.0


def papg(X, ybar, gamma, L, K, Tprev=None, Tt=None, t=1.0, nthreads=0, inplace=False):
    """Run K P-APG iterations (Fig. 2) from state (theta^{k-1}, theta~^k, t_k).

    Defaults are the paper's start: theta^0 = 0, theta~^1 = theta^0, t_1 = 1.
    Returns dict(Tprev=theta^{last}, Tt=theta~^{last+1}, t=t_{last+1}, y, xi) where
    (y, xi) = eta of the last iteration's Step 1.
    inplace=True: Tprev and Tt (C-contiguous float64 N x N, both given) are updated in place
    instead of copied -- memory only (full-size C5 states are 32 GiB each); same arithmetic.
    """
    X = _c64(X)
    ybar = _c64(ybar)
    N, n = X.shape
    if inplace:
        for a in (Tprev, Tt):
            if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.c_contiguous
                    and a.shape == (N, N)):
                raise ValueError("inplace=True needs C-contiguous float64 N x N Tprev and Tt")
    else:
        Tprev = np.zeros((N, N)) if Tprev is None else _c64(Tprev).copy()
        Tt = Tprev.copy() if Tt is None else _c64(Tt).copy()
    y = np.zeros(N)
    xi = np.zeros((N, n))
    tt = C.c_double(float(t))
    rc = lib().oracle_papg(N, n, X, ybar, float(gamma), float(L), int(K), Tprev, Tt, C.byref(tt),
                           y.ctypes.data, xi.ctypes.data, int(nthreads))
    if rc:
        raise MemoryError("oracle_papg allocation failed")
    return dict(Tprev=Tprev, Tt=Tt, t=tt.value, y=y, xi=xi)


def papg_adaptive(X, ybar, gamma, s, K, ups=2.0, Tprev=None, Tt=None, t=1.0, max_trials=200, backtrack=False,
                  nthreads=0):
    """K iterations of P-APG with the adaptive step rule of P:400-407 from state
    (theta^{k-1}, theta~^k, t_k, s_{k-1}); the paper's start is theta^0 = 0, t_1 = 1, s_0 = L.

    Returns dict(Tprev, Tt, t, s, trials (l_k + 1 per iteration), s_hist (s_k), y, xi)."""
    X = _c64(X)
    ybar = _c64(ybar)
    N, n = X.shape
    Tprev = np.zeros((N, N)) if Tprev is None else _c64(Tprev).copy()
    Tt = Tprev.copy() if Tt is None else _c64(Tt).copy()
    y = np.zeros(N)
    xi = np.zeros((N, n))
    trials = np.zeros(max(int(K), 1), dtype=np.int64)
    s_hist = np.zeros(max(int(K), 1))
    tt, ss = C.c_double(float(t)), C.c_double(float(s))
    rc = lib().oracle_papg_adaptive(N, n, X, ybar, float(gamma), float(ups), int(K), Tprev, Tt, C.byref(tt),
                                    C.byref(ss), trials, s_hist, y.ctypes.data, xi.ctypes.data, int(max_trials),
                                    1 if backtrack else 0, int(nthreads))
    if rc == 1:
        raise MemoryError("oracle_papg_adaptive allocation failed")
    if rc == 2:
        raise RuntimeError("adaptive step: no l_k <= max_trials passed Eq. (adaptive-check)")
    return dict(Tprev=Tprev, Tt=Tt, t=tt.value, s=ss.value, trials=trials[:K], s_hist=s_hist[:K], y=y, xi=xi)


def continuation(X, ybar, sigma2, eps0, beta, kappa_gamma, iters, Theta0=None, stop=None, ups=None, nthreads=0):
    """Continuation over gamma (Section 2.4.1): for outer t = 1..T,
        eps_t = eps0 / beta^t,  gamma_t = kappa_gamma eps_t,  L_t = sigma2 / gamma_t  (Eq. (lischitz)),
    theta^(t) = P-APG (Fig. 2) on the gamma_t problem started from theta^(t-1) (theta~^1 = theta^0
    = theta^(t-1), t_1 = 1), theta^(0) = Theta0 (default 0), run for iters[t-1] iterations
    (the a-priori budget K_t of P:580 is the caller's), or fewer when ``stop`` = (m, infeas_tol,
    gap_tol) holds at a multiple of m: normalized infeasibility <= infeas_tol and |gap| / (N^2 - N)
    <= gap_tol at eta(theta^k) (the stopping pair of P:1106).  ups: use the adaptive step rule
     inside the stages with growth factor ups, s_0 = L_t at each stage start.

    Returns a list with one dict per stage: gamma, L, iters, Theta, y, xi (= eta(theta^(t)))."""
    X = _c64(X)
    ybar = _c64(ybar)
    N, n = X.shape
    Th = np.zeros((N, N)) if Theta0 is None else _c64(Theta0).copy()
    out = []
    for t, K in enumerate(iters, start=1):
        gamma = kappa_gamma * eps0 / beta ** t
        L = sigma2 / gamma
        st = dict(Tprev=Th, Tt=Th, t=1.0, s=L)
        done = 0
        while done < K:
            m = K - done if stop is None else min(stop[0], K - done)
            if ups is None:
                st = papg(X, ybar, gamma, L, m, Tprev=st["Tprev"], Tt=st["Tt"], t=st["t"], nthreads=nthreads)
            else:
                st = papg_adaptive(X, ybar, gamma, st["s"], m, ups=ups, Tprev=st["Tprev"], Tt=st["Tt"], t=st["t"],
                                   nthreads=nthreads)
            done += m
            if stop is not None:
                y, xi = eta(X, ybar, gamma, st["Tprev"], nthreads)
                sd = stats(X, ybar, gamma, st["Tprev"], y, xi, nthreads)
                if sd["infeas_norm"] <= stop[1] and abs(sd["gap"]) / (N * N - N) <= stop[2]:
                    break
        Th = st["Tprev"]
        y, xi = eta(X, ybar, gamma, Th, nthreads)
        out.append(dict(gamma=gamma, L=L, iters=done, Theta=Th.copy(), y=y, xi=xi))
    return out


def eta(X, ybar, gamma, T, nthreads=0):
    """eta(Theta) = Step-1 minimizer at Theta (Theorem 1); returns (y, xi)."""
    X = _c64(X)
    N, n = X.shape
    y = np.zeros(N)
    xi = np.zeros((N, n))
    rc = lib().oracle_eta(N, n, X, _c64(ybar), float(gamma), _c64(T), y, xi, int(nthreads))
    if rc:
        raise MemoryError("oracle_eta allocation failed")
    return y, xi


def stats(X, ybar, gamma, T, y, xi, nthreads=0):
    """dict(r_gamma, g, gap, max_violation, infeas_norm) -- see papg_oracle.c oracle_stats."""
    X = _c64(X)
    N, n = X.shape
    out = np.zeros(5)
    Tp = None if T is None else _c64(T)
    rc = lib().oracle_stats(N, n, X, _c64(ybar), float(gamma), None if Tp is None else Tp.ctypes.data,
                            _c64(y), _c64(xi).reshape(N, n), out, int(nthreads))
    if rc:
        raise MemoryError("oracle_stats allocation failed")
    return dict(r_gamma=out[0], g=out[1], gap=out[2], max_violation=out[3], infeas_norm=out[4])


def project_rows(X, y, xi, L, rows, Tt_rows, nthreads=0):
    """Step 2 for selected rows given eta^k and the rows of theta~^k."""
    X = _c64(X)
    N, n = X.shape
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    out = np.zeros((len(rows), N))
    lib().oracle_project_rows(N, n, X, _c64(y), _c64(xi).reshape(N, n), float(L), rows, len(rows),
                              _c64(Tt_rows).reshape(len(rows), N), out, int(nthreads))
    return out


def extrapolate(Tk, Tkm1, t_k, t_kp1):
    """Step 4 of Fig. 2: theta~^{k+1} = theta^k + ((t_k - 1)/t_{k+1}) (theta^k - theta^{k-1})."""
    Tk = _c64(Tk)
    return Tk + ((t_k - 1.0) / t_kp1) * (Tk - _c64(Tkm1))


def state_after(X, ybar, gamma, L, K, nthreads=0):
    """Oracle run of K >= 1 iterations from theta^0 = 0 returning the GPU-style state
    (Theta^K, Theta^{K-1}, t_K, t_{K+1}) plus eta^K (Step 1 of iteration K)."""
    a = papg(X, ybar, gamma, L, K - 1, nthreads=nthreads)          # Tprev = theta^{K-1}, t = t_K
    b = papg(X, ybar, gamma, L, 1, Tprev=a["Tprev"], Tt=a["Tt"], t=a["t"], nthreads=nthreads)
    return dict(Tk=b["Tprev"], Tkm1=a["Tprev"], t_k=a["t"], t_kp1=b["t"], y=b["y"], xi=b["xi"])
