"""GPU parity of the continuation over gamma (Section 2.4.1) and of cr_set_gamma
(restart of Fig. 2 at the current iterate) through the C ABI vs the fp64 oracle."""
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


@pytest.mark.parametrize("N,n,prec,kernel,iters,tol", [
    (120, 3, "fp64", "auto", [25, 25, 25], 1e-11),
    (1000, 20, "fp32", "tc", [40, 40], 1e-4),
])
def test_continuation_matches_oracle(crp, N, n, prec, kernel, iters, tol):
    X, ybar = crdata.random_problem(N, n, seed=11, fp32=prec == "fp32")
    gamma0 = 1e-2
    L0 = ref.lipschitz(X, gamma0)
    sigma2 = L0 * gamma0                      # both sides use sigma_max(C)^2 = L0 gamma0
    want = oracle.continuation(X, ybar, sigma2, eps0=1e-1, beta=4.0, kappa_gamma=0.1, iters=iters)
    s = crp.Solver(X, ybar, gamma0, L=L0, prec=prec, kernel=kernel)
    rep = s.continuation(1e-1, 4.0, 0.1, iters)
    assert rep["stages_run"] == len(iters) and rep["iters_total"] == sum(iters)
    assert rep["gamma_last"] == want[-1]["gamma"]
    assert rep["L_last"] == pytest.approx(want[-1]["L"], rel=1e-15)
    T = s.get_theta()[0]
    assert rel(T, want[-1]["Theta"]) <= tol
    y, xi, st = s.primal()
    assert rel(y, want[-1]["y"]) <= tol and rel(xi, want[-1]["xi"]) <= tol
    so = oracle.stats(X, ybar, want[-1]["gamma"], want[-1]["Theta"], want[-1]["y"], want[-1]["xi"])
    assert abs(st["r_gamma"] - so["r_gamma"]) <= max(tol, 1e-12) * abs(so["r_gamma"])
    s.close()


def test_continuation_stagewise_and_adaptive(crp):
    """Stage by stage (cr_set_gamma + cr_solve) equals the oracle after every stage, with the
    adaptive rule inside the stages (s_0 = L_t at each restart)."""
    N, n = 90, 2
    X, ybar = crdata.random_problem(N, n, seed=12)
    gamma0 = 5e-2
    L0 = ref.lipschitz(X, gamma0)
    iters = [15, 15, 15]
    want = oracle.continuation(X, ybar, L0 * gamma0, eps0=0.2, beta=3.0, kappa_gamma=0.5, iters=iters, ups=2.0)
    s = crp.Solver(X, ybar, gamma0, L=L0, prec="fp64", adaptive=True)
    s.set_step_rule("adaptive", 2.0)
    for t, (K, w) in enumerate(zip(iters, want), start=1):
        s.set_gamma(0.5 * 0.2 / 3.0 ** t)
        assert s.step_info()["s"] == pytest.approx(w["L"], rel=1e-15)
        s.solve(K)
        assert rel(s.get_theta()[0], w["Theta"]) <= 1e-11, t
    s.close()


def test_set_gamma_restarts_fig2(crp):
    """cr_set_gamma(g, L): the next step is Fig. 2's first iteration from theta^0 = current Theta^k
    (theta~^1 = theta^0, t_1 = 1) on the new problem."""
    N, n = 300, 5
    X, ybar = crdata.random_problem(N, n, seed=13)
    g0, g1 = 1e-2, 3e-3
    L0, L1 = ref.lipschitz(X, g0), ref.lipschitz(X, g1)
    s = crp.Solver(X, ybar, g0, L=L0, prec="fp64")
    s.solve(30)
    T30 = s.get_theta()[0]
    s.set_gamma(g1, L1)
    assert s.L == L1
    s.step()
    T, T1, tk, tk1 = s.get_theta()
    o30 = oracle.papg(X, ybar, g0, L0, 30)["Tprev"]                 # the oracle's own theta^30
    want = oracle.papg(X, ybar, g1, L1, 1, Tprev=o30, Tt=o30, t=1.0)
    assert rel(T, want["Tprev"]) <= 1e-11
    np.testing.assert_array_equal(T1, T30)
    assert tk1 == oracle.momentum_next(1.0)
    with pytest.raises(crp.CrError):
        s.set_gamma(-1.0)
    with pytest.raises(crp.CrError):
        s.set_gamma(2.0)                       # L from sigma^2 / gamma needs gamma <= 1
    s.close()
