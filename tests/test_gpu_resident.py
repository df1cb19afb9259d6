"""The SMEM-resident small-N solver (kernels/resident.cu): K constant-step P-APG iterations
(Fig. 2) in one cooperative launch with both state matrices in shared memory.
cr_solve picks it for world == 1, n <= 32, row-major (SIMT-layout) configs -- C1 and C2."""
import numpy as np
import pytest

import crdata
import oracle
from oracle import ref

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


@pytest.fixture(scope="module")
def crp():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1608_02227_b200 import build
    build.build()
    import paper_1608_02227_b200 as m
    return m


@pytest.mark.parametrize("N,n,prec,K,tol", [
    (50, 2, "fp64", 120, 1e-12),         # C1 shape (one CTA)
    (300, 5, "fp64", 60, 1e-12),
    (1000, 10, "fp32", 100, 1e-5),       # C2 shape (148 CTAs, grid syncs)
    (129, 15, "fp32", 40, 1e-5),         # widest fp32 SIMT-layout n
    (777, 3, "fp32", 50, 1e-5),          # ragged CTA row ranges
])
def test_resident_matches_oracle(crp, N, n, prec, K, tol):
    X, ybar = crdata.random_problem(N, n, seed=N + n, fp32=prec == "fp32")
    gamma = 1e-3
    L = ref.lipschitz(X, gamma)
    want = oracle.papg(X, ybar, gamma, L, K)
    s = crp.Solver(X, ybar, gamma, L=L, prec=prec)
    l0 = s.launch_count
    s.solve(K)
    assert s.launch_count - l0 == 1                      # one cooperative launch for all K
    T, T1, tk, tk1 = s.get_theta()
    assert np.all(T >= 0) and np.all(np.diag(T) == 0)
    assert rel(T, want["Tprev"]) <= (tol if prec == "fp64" else 1e-4)
    assert tk1 == want["t"]
    y, xi = s.get_eta()                                  # eta^K = Step 1 of iteration K
    assert rel(y, want["y"]) <= tol and rel(xi, want["xi"]) <= max(tol, 1e-9 if prec == "fp64" else 1e-5)
    yo, xio = oracle.eta(X, ybar, gamma, want["Tprev"])
    so = oracle.stats(X, ybar, gamma, want["Tprev"], yo, xio)
    _, _, sg = s.primal()
    assert abs(sg["r_gamma"] - so["r_gamma"]) <= 1e-5 * abs(so["r_gamma"])
    s.close()


def test_resident_deterministic_chunked_and_continues_streaming(crp):
    X, ybar = crdata.random_problem(700, 6, seed=9, fp32=True)
    gamma = 1e-3
    L = ref.lipschitz(X, gamma)
    a = crp.Solver(X, ybar, gamma, L=L)
    a.solve(37)
    b = crp.Solver(X, ybar, gamma, L=L)
    b.solve(20)
    b.solve(17)
    np.testing.assert_array_equal(a.get_theta()[0], b.get_theta()[0])
    np.testing.assert_array_equal(a.get_theta()[1], b.get_theta()[1])
    # the state it leaves is the streaming path's: a further cr_dual_step continues Fig. 2
    a.step()
    want = oracle.papg(X, ybar, gamma, L, 38)
    assert rel(a.get_theta()[0], want["Tprev"]) <= 1e-4
    # with stop tests every 10 iterations (chunks of 10 launches)
    c = crp.Solver(X, ybar, gamma, L=L)
    rep = c.solve(37, report_every=10, infeas_tol=0.0, gap_tol=0.0)
    assert rep["iters"] == 37 and not rep["converged"]
    np.testing.assert_array_equal(c.get_theta()[0], b.get_theta()[0])
    for s in (a, b, c):
        s.close()
