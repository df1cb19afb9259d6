"""GPU parity of the adaptive step rule (PAPG_A) through the C ABI vs the fp64 oracle.

The oracle evaluates Eq. (adaptive-check) literally (g values and the gradient inner product);
libcr evaluates the identical inequality in its quadratic form (R15, pinned by
tests/test_oracle_pins.py::test_adaptive_quadratic_identity).  Accept/reject decisions are
integers decided by floating point: the cases below stay in the early iterations, where the
check margins are far above either side's rounding, and compare the decisions exactly.
"""
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


def rnd32(a):
    return np.asarray(a, dtype=np.float64).astype(np.float32).astype(np.float64)


@pytest.fixture(scope="module")
def crp():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1608_02227_b200 import build
    build.build()
    import paper_1608_02227_b200 as m
    return m


@pytest.mark.parametrize("N,n,K,prec,kernel,tol", [
    (50, 2, 40, "fp64", "auto", 1e-11),        # C1 shape, SIMT fp64
    (97, 3, 30, "fp64", "auto", 1e-11),        # ragged tiles
    (300, 5, 15, "fp32", "simt", 2e-5),        # (its fp32-storage floor grows 8e-5 by K=25: tests/numerics/fp32_storage_floor_adaptive.py)
    (1000, 20, 25, "fp32", "tc", 2e-5),        # tcgen05 pass, several 128-row blocks, ragged tail
    (700, 40, 20, "fp32", "tc", 2e-5),
])
def test_adaptive_run_matches_oracle(crp, N, n, K, prec, kernel, tol):
    X, ybar = crdata.random_problem(N, n, seed=N + n, fp32=prec == "fp32")
    gamma = 1e-3
    L = ref.lipschitz(X, gamma)
    want = oracle.papg_adaptive(X, ybar, gamma, L, K, ups=2.0)
    s = crp.Solver(X, ybar, gamma, L=L, prec=prec, kernel=kernel, adaptive=True)
    s.set_step_rule("adaptive", 2.0)
    trials, shist = [], []
    for _ in range(K):
        s.step()
        info = s.step_info()
        trials.append(info["trials_last"])
        shist.append(info["s"])
    np.testing.assert_array_equal(trials, want["trials"])
    np.testing.assert_allclose(shist, want["s_hist"], rtol=1e-15)
    T, _, _, t_next = s.get_theta()
    assert np.all(T >= 0) and np.all(np.diag(T) == 0)
    assert rel(T, want["Tprev"]) <= tol, rel(T, want["Tprev"])
    assert t_next == want["t"]                 # t_{K+1}, the momentum scalar the next step uses
    assert s.step_info()["trials_total"] == int(np.sum(want["trials"]))
    s.close()


@pytest.mark.parametrize("N,n,prec,kernel", [(200, 4, "fp64", "auto"), (600, 24, "fp32", "tc")])
def test_adaptive_single_step_from_oracle_state(crp, N, n, prec, kernel):
    """Mid-run state of the oracle's adaptive run -> one GPU adaptive step from it."""
    X, ybar = crdata.random_problem(N, n, seed=7, fp32=prec == "fp32")
    gamma = 1e-3
    L = ref.lipschitz(X, gamma)
    a = oracle.papg_adaptive(X, ybar, gamma, L, 14)
    b = oracle.papg_adaptive(X, ybar, gamma, a["s"], 1, Tprev=a["Tprev"], Tt=a["Tt"], t=a["t"])
    r = (lambda v: v) if prec == "fp64" else rnd32
    Tk, Tkm1 = r(b["Tprev"]), r(a["Tprev"])
    t_k, t_kp1 = a["t"], b["t"]
    Tt = oracle.extrapolate(Tk, Tkm1, t_k, t_kp1)
    want = oracle.papg_adaptive(X, ybar, gamma, b["s"], 1, Tprev=Tk, Tt=Tt, t=t_kp1)
    s = crp.Solver(X, ybar, gamma, L=L, prec=prec, kernel=kernel, adaptive=True)
    s.set_theta(Tk, Tkm1, t_k, t_kp1)
    s.set_step_rule("adaptive", 2.0, s_prev=b["s"])
    s.step()
    info = s.step_info()
    assert info["trials_last"] == want["trials"][0]
    assert info["s"] == want["s_hist"][0]
    T, T1, _, _ = s.get_theta()
    y, xi = s.get_eta()
    tol = 1e-12 if prec == "fp64" else 1e-5
    assert rel(T, want["Tprev"]) <= tol
    np.testing.assert_array_equal(T1, Tk)
    assert rel(y, want["y"]) <= tol and rel(xi, want["xi"]) <= tol
    s.close()


@pytest.mark.parametrize("N,n,prec,kernel", [(300, 5, "fp64", "auto"), (900, 20, "fp32", "tc")])
def test_rejected_trials_leave_state_intact(crp, N, n, prec, kernel):
    """ups = 1e30: the l = 0 trial (step 1e30/s) is always rejected and l = 1 (s = L) accepted, so
    every iteration writes and discards one trial Theta^k; the accepted iterates must equal the
    constant-step path's bit for bit (the rejected trial never touched Theta^{k-1}, Theta^{k-2})."""
    X, ybar = crdata.random_problem(N, n, seed=3, fp32=prec == "fp32")
    gamma = 1e-3
    a = crp.Solver(X, ybar, gamma, prec=prec, kernel=kernel, adaptive=True)
    a.set_step_rule("adaptive", 1e30)
    c = crp.Solver(X, ybar, gamma, prec=prec, kernel=kernel)
    for _ in range(12):
        a.step()
        assert a.step_info()["trials_last"] == 2
        c.step()
    Ta, Ta1, ta, ta1 = a.get_theta()
    Tc, Tc1, tc, tc1 = c.get_theta()
    np.testing.assert_array_equal(Ta, Tc)
    np.testing.assert_array_equal(Ta1, Tc1)
    assert (ta, ta1) == (tc, tc1)
    # switching back to the constant rule continues from the same state (graph path)
    a.set_step_rule("constant")
    a.solve(5)
    c.solve(5)
    np.testing.assert_array_equal(a.get_theta()[0], c.get_theta()[0])
    a.close()
    c.close()


def test_adaptive_needs_third_buffer(crp):
    X, ybar = crdata.random_problem(100, 3, seed=1)
    s = crp.Solver(X, ybar, 1e-3)
    with pytest.raises(crp.CrError):
        s.set_step_rule("adaptive", 2.0)
    s2 = crp.Solver(X, ybar, 1e-3, adaptive=True)
    with pytest.raises(crp.CrError):
        s2.set_step_rule("adaptive", 1.0)          # upsilon must be > 1
    s.close()
    s2.close()


@pytest.mark.parametrize("N,n,prec,kernel", [(97, 3, "fp64", "auto"), (1000, 20, "fp32", "tc")])
def test_adaptive_graph_solve_equals_stepwise(crp, N, n, prec, kernel, monkeypatch):
    """cr_solve runs each adaptive iteration as one CUDA graph (a WHILE node over trials, the
    accept/retry decision on the device); it must reproduce the host-driven trial loop of
    cr_dual_step bit for bit, decisions and counters included."""
    X, ybar = crdata.random_problem(N, n, seed=31, fp32=prec == "fp32")
    gamma = 1e-3
    L = ref.lipschitz(X, gamma)
    a = crp.Solver(X, ybar, gamma, L=L, prec=prec, kernel=kernel, adaptive=True)
    b = crp.Solver(X, ybar, gamma, L=L, prec=prec, kernel=kernel, adaptive=True)
    for s in (a, b):
        s.set_step_rule("adaptive", 2.0)
    a.solve(15)
    for _ in range(15):
        b.step()
    np.testing.assert_array_equal(a.get_theta()[0], b.get_theta()[0])
    np.testing.assert_array_equal(a.get_theta()[1], b.get_theta()[1])
    ia, ib = a.step_info(), b.step_info()
    assert ia == ib
    want = oracle.papg_adaptive(X, ybar, gamma, L, 15)
    assert ia["trials_total"] == int(np.sum(want["trials"])) and ia["s"] == want["s_hist"][-1]
    a.close()
    b.close()


@pytest.mark.parametrize("N,n,prec,kernel", [(120, 3, "fp64", "auto"), (1000, 20, "fp32", "tc")])
def test_backtrack_variant_matches_oracle(crp, N, n, prec, kernel):
    """CR_STEP_BACKTRACK (monotone, R18) from s_0 = L/64: same decisions as the oracle."""
    X, ybar = crdata.random_problem(N, n, seed=N + 7, fp32=prec == "fp32")
    gamma = 1e-3
    L = ref.lipschitz(X, gamma)
    K = 25
    want = oracle.papg_adaptive(X, ybar, gamma, L / 64, K, backtrack=True)
    s = crp.Solver(X, ybar, gamma, L=L, prec=prec, kernel=kernel, adaptive=True)
    s.set_step_rule("backtrack", 2.0, s_prev=L / 64)
    trials = []
    for _ in range(K):
        s.step()
        trials.append(s.step_info()["trials_last"])
    np.testing.assert_array_equal(trials, want["trials"])
    assert s.step_info()["s"] == want["s"]
    assert rel(s.get_theta()[0], want["Tprev"]) <= (1e-11 if prec == "fp64" else 2e-5)
    s.close()
