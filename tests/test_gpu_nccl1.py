"""The NCCL code path on one GPU: with CR_FORCE_NCCL a single rank still runs every collective
(all-gather of y', reduce-scatter of the column sums, scalar all-reduces) through a 1-rank NCCL
communicator, captured in the CUDA graphs like a multi-GPU run.  With one rank every collective
is a copy, so the iterates must equal the collective-free path bit for bit."""
import numpy as np
import pytest

import crdata
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


@pytest.mark.parametrize("N,n,prec,kernel", [(300, 5, "fp64", "auto"), (1000, 20, "fp32", "tc"), (517, 6, "fp32", "simt")])
def test_forced_nccl_equals_collective_free(crp, N, n, prec, kernel, monkeypatch):
    X, ybar = crdata.random_problem(N, n, seed=41, fp32=prec == "fp32")
    gamma = 1e-3
    L = ref.lipschitz(X, gamma)
    monkeypatch.setenv("CR_NO_RESIDENT", "1")       # the streaming path on both sides
    b = crp.Solver(X, ybar, gamma, L=L, prec=prec, kernel=kernel)
    monkeypatch.setenv("CR_FORCE_NCCL", "1")
    a = crp.Solver(X, ybar, gamma, L=L, prec=prec, kernel=kernel)
    for s in (a, b):
        s.solve(20)                                  # graph replay (NCCL calls captured)
        s.step()                                     # eager
    np.testing.assert_array_equal(a.get_theta()[0], b.get_theta()[0])
    np.testing.assert_array_equal(a.get_sums(0)[1], b.get_sums(0)[1])
    ya, xia, sa = a.primal()
    yb, xib, sb = b.primal()
    np.testing.assert_array_equal(ya, yb)
    np.testing.assert_array_equal(xia, xib)
    assert sa == sb
    Z = np.random.default_rng(0).standard_normal((17, n))
    np.testing.assert_array_equal(a.predict(Z), b.predict(Z))
    rep = a.solve(10, report_every=5, infeas_tol=0.0, gap_tol=0.0)
    assert rep["iters"] == 10
    a.close()
    b.close()


def test_forced_nccl_adaptive(crp, monkeypatch):
    X, ybar = crdata.random_problem(400, 4, seed=42)
    gamma = 1e-3
    L = ref.lipschitz(X, gamma)
    b = crp.Solver(X, ybar, gamma, L=L, prec="fp64", adaptive=True)
    monkeypatch.setenv("CR_FORCE_NCCL", "1")
    a = crp.Solver(X, ybar, gamma, L=L, prec="fp64", adaptive=True)
    for s in (a, b):
        s.set_step_rule("adaptive", 2.0)
        s.solve(12)
    np.testing.assert_array_equal(a.get_theta()[0], b.get_theta()[0])
    assert a.step_info() == b.step_info()
    a.close()
    b.close()
