"""GPU parity of cr_predict, the max-affine estimator f_hat(z) = max_i y_i + xi_i^T (z - x_i) at
eta(Theta^k) (Theorem 1), against oracle/ref.predict (the definition)."""
import threading

import numpy as np
import pytest

import crdata
import oracle
from oracle import ref

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def crp():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1608_02227_b200 import build
    build.build()
    import paper_1608_02227_b200 as m
    return m


@pytest.mark.parametrize("N,n,M,prec,kernel", [(200, 3, 333, "fp64", "auto"), (1000, 20, 70, "fp32", "tc"),
                                               (130, 80, 5, "fp32", "tc")])
def test_predict_matches_definition(crp, N, n, M, prec, kernel):
    X, ybar = crdata.random_problem(N, n, seed=21, fp32=prec == "fp32")
    gamma = 1e-3
    L = ref.lipschitz(X, gamma)
    s = crp.Solver(X, ybar, gamma, L=L, prec=prec, kernel=kernel)
    s.solve(40)
    Z = np.random.default_rng(1).standard_normal((M, n))
    # at random points and at the data points, with the oracle's eta after the same iterations
    want = oracle.papg(X, ybar, gamma, L, 40)
    yo, xio = oracle.eta(X, ybar, gamma, want["Tprev"])
    tol = 1e-10 if prec == "fp64" else 1e-4
    np.testing.assert_allclose(s.predict(Z), ref.predict(X, yo, xio, Z), rtol=tol, atol=tol)
    np.testing.assert_allclose(s.predict(X[:50]), ref.predict(X, yo, xio, X[:50]), rtol=tol, atol=tol)
    s.close()


def test_predict_sharded_local_group(crp):
    import torch
    N, n, M, world = 301, 4, 100, 3
    X, ybar = crdata.random_problem(N, n, seed=22)
    gamma = 1e-3
    L = ref.lipschitz(X, gamma)
    Z = np.random.default_rng(2).standard_normal((M, n))
    g = crp.LocalGroup(world)
    out = [None] * world

    def body(r):
        torch.cuda.set_device(0)
        st = torch.cuda.Stream()
        sol = crp.Solver(X, ybar, gamma, L=L, prec="fp64", group=g, rank=r, stream=st)
        sol.solve(25)
        out[r] = sol.predict(Z)
        sol.close()

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    g.close()
    want = oracle.papg(X, ybar, gamma, L, 25)
    yo, xio = oracle.eta(X, ybar, gamma, want["Tprev"])
    for r in range(world):
        np.testing.assert_array_equal(out[r], out[0])
    np.testing.assert_allclose(out[0], ref.predict(X, yo, xio, Z), rtol=1e-10, atol=1e-10)
