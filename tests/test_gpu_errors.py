"""Error behaviour of the C ABI (include/cr.h conventions): CR_ERR_INVALID_ARG leaves the context
usable and unchanged; bad shapes and values are rejected before any device work."""
import ctypes as C

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


def test_invalid_arguments_leave_context_usable(crp):
    X, ybar = crdata.random_problem(200, 4, seed=51)
    L = ref.lipschitz(X, 1e-3)
    s = crp.Solver(X, ybar, 1e-3, L=L, adaptive=True)
    s.solve(5)
    T5 = s.get_theta()[0]
    bad = np.zeros((200, 200))
    bad[3, 7] = -1.0                                   # negative multiplier
    with pytest.raises(crp.CrError, match="INVALID_ARG"):
        s.set_theta(bad, None)
    bad[3, 7] = 0.0
    bad[5, 5] = 1.0                                    # nonzero diagonal
    with pytest.raises(crp.CrError, match="INVALID_ARG"):
        s.set_theta(bad, None)
    with pytest.raises(crp.CrError, match="INVALID_ARG"):
        s.set_theta(None, None, t_km1=0.5)             # t < 1
    with pytest.raises(crp.CrError, match="INVALID_ARG"):
        s.set_step_rule("adaptive", 0.9)
    with pytest.raises(crp.CrError, match="INVALID_ARG"):
        s.set_gamma(0.0)
    with pytest.raises(crp.CrError, match="INVALID_ARG"):
        s.continuation(1e-1, 0.5, 1.0, [10])           # beta <= 1
    with pytest.raises(crp.CrError, match="INVALID_ARG"):
        s.predict(np.array([[np.nan, 0, 0, 0]]))
    with pytest.raises(crp.CrError, match="INVALID_ARG"):
        s.get_theta_rows(0, 190, 20)                   # past the shard
    st = s.lib.cr_solve(s.h, -1, None, None)
    assert st == crp.binding.CR_ERR_INVALID_ARG
    # the context is unchanged and still iterates like the oracle
    np.testing.assert_array_equal(s.get_theta()[0], T5)
    s.solve(5)
    want = oracle.papg(X, ybar, 1e-3, L, 10)
    assert np.linalg.norm(s.get_theta()[0] - want["Tprev"]) <= 1e-5 * np.linalg.norm(want["Tprev"])
    s.close()


def test_init_rejects_bad_problems(crp):
    lib = crp.load()
    X, ybar = crdata.random_problem(64, 3, seed=52)
    for N, n, gamma in ((1, 3, 1e-3), (64, 0, 1e-3), (64, 3, -1.0), (64, 500, 1e-3)):
        assert crp.workspace_size(max(N, 2), max(n, 1)) > 0 or n == 500
    Xn = X.copy()
    Xn[0, 0] = np.nan
    with pytest.raises(crp.CrError):
        crp.Solver(Xn, ybar, 1e-3)
    with pytest.raises(crp.CrError):
        crp.Solver(X, ybar, 2.0)                       # gamma > 1 with L computed (R4)
    with pytest.raises(crp.CrError):
        crp.Solver(X, ybar, 1e-3, prec="fp64", kernel="tc")   # tcgen05 pass is fp32 only
    assert lib.cr_init(None, C.byref(C.c_void_p())) == crp.binding.CR_ERR_INVALID_ARG


@pytest.mark.parametrize("path", ["graph", "host_step", "graph_with_stop"])
def test_exhausted_adaptive_trials_poison_the_context(crp, path):
    """an adaptive iteration whose trials l = 0..63 all fail Eq. (adaptive-check)
     leaves no valid iterate (t_k not advanced, the spare buffer holds a rejected trial):
    the call returns CR_ERR_STATE and the context is poisoned -- every later call is refused, on
    the CUDA-graph path (cr_solve, checked at its end or at its stop tests) and the host path
    (cr_dual_step) alike.  Forced with s_prev far below the curvature and upsilon close to 1, so
    s_{k-1} upsilon^(l-1) never reaches the passing range in 64 trials."""
    X, ybar = crdata.random_problem(300, 4, seed=52, fp32=True)
    L = ref.lipschitz(X, 1e-3)
    s = crp.Solver(X, ybar, 1e-3, L=L, adaptive=True)
    s.set_step_rule("adaptive", 1.01, L * 1e-12)
    with pytest.raises(crp.CrError, match="adaptive"):
        if path == "graph":
            s.solve(4)
        elif path == "graph_with_stop":
            s.solve(6, report_every=2)
        else:
            s.step()
    with pytest.raises(crp.CrError):
        s.step()
    with pytest.raises(crp.CrError):
        s.get_theta()
    s.close()
