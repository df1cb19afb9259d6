"""Pins for the fp64 oracle (oracle/) against what the paper and mathematics fix.

Each test names the pin of SURVEY.md §8(c) / DESIGN.md §Oracle it implements.
None of these tests touch the GPU path.
"""
import json
import math
import os

import numpy as np
import pytest

import crdata
import oracle
from oracle import ref

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _tiny(N, n, seed=0, noise=0.3):
    return crdata.random_problem(N, n, seed=seed, noise_sd=noise)


# ---------------------------------------------------------------- P2 operators
def test_spec_worked_operator_values():
    """SPEC.md S:51, S:61, S:69 worked values for the dense Def. A1A2 construction."""
    g = _gold("spec_operator_examples.json")
    A1 = ref.dense_A1(2)
    np.testing.assert_array_equal(A1 @ np.array(g["A1_y"]["y"]), g["A1_y"]["expect"])
    np.testing.assert_array_equal(A1.T @ np.array(g["A1T_z"]["z"]), g["A1T_z"]["expect"])
    A2 = ref.dense_A2(np.array(g["A2_xi"]["X"]))
    np.testing.assert_array_equal(A2 @ np.array(g["A2_xi"]["xi"]), g["A2_xi"]["expect"])


@pytest.mark.parametrize("N,n", [(3, 1), (5, 2), (7, 3)])
def test_dense_rows_are_pair_constraints(N, n):
    """Row (l1,l2) of A1 y + A2 xi equals y_l2 - y_l1 + xi_l1^T (x_l1 - x_l2) (Eq. (original))."""
    X, _ = _tiny(N, n, seed=N)
    rng = np.random.default_rng(1)
    y, xi = rng.standard_normal(N), rng.standard_normal((N, n))
    z = ref.dense_A1(N) @ y + ref.dense_A2(X) @ xi.reshape(-1)
    for i in range(N):
        for j in range(N):
            if i != j:
                want = y[j] - y[i] + xi[i] @ (X[i] - X[j])
                assert abs(z[ref.pair_index(i, j, N)] - want) < 1e-12


@pytest.mark.parametrize("N,n,seed", [(4, 1, 0), (6, 2, 1), (8, 3, 2)])
def test_oracle_eta_equals_dense_stationary_point(N, n, seed):
    """Step 1 closed form in the C oracle == dense G^{-1} C^T theta + (ybar, 0)."""
    X, ybar = _tiny(N, n, seed)
    T = crdata.random_theta(N, seed=seed + 10)
    gamma = 0.05
    y, xi = oracle.eta(X, ybar, gamma, T)
    yd, xid = ref.eta_dense(ref.theta_vec(T), X, ybar, gamma)
    np.testing.assert_allclose(y, yd, rtol=0, atol=1e-12)
    np.testing.assert_allclose(xi, xid, rtol=0, atol=1e-11)
    # and it really is the minimizer: gradient of the Lagrangian vanishes
    th = ref.theta_vec(T)
    base = ref.lagrangian_dense(y, xi, th, X, ybar, gamma)
    rng = np.random.default_rng(seed)
    for _ in range(5):
        dy, dxi = rng.standard_normal(N) * 1e-3, rng.standard_normal((N, n)) * 1e-3
        assert ref.lagrangian_dense(y + dy, xi + dxi, th, X, ybar, gamma) >= base - 1e-14


@pytest.mark.parametrize("N,n,seed", [(4, 1, 3), (6, 2, 4), (8, 3, 5)])
def test_oracle_step_equals_dense_fig2_step(N, n, seed):
    """One Fig. 2 iteration from a random mid-run state vs dense Steps 1-4."""
    X, ybar = _tiny(N, n, seed)
    gamma, L = 0.02, 37.0
    Tprev = crdata.random_theta(N, seed=seed, scale=0.1)
    Tt = crdata.random_theta(N, seed=seed + 1, scale=0.1)
    t = 2.7
    out = oracle.papg(X, ybar, gamma, L, 1, Tprev=Tprev, Tt=Tt, t=t)
    # dense reference
    th_t = ref.theta_vec(Tt)
    y, xi = ref.eta_dense(th_t, X, ybar, gamma)
    Ceta = ref.dense_C(X) @ np.concatenate([y, xi.reshape(-1)])
    th_k = np.maximum(0.0, th_t - Ceta / L)
    tn = (1 + math.sqrt(1 + 4 * t * t)) / 2
    th_next = th_k + (t - 1) / tn * (th_k - ref.theta_vec(Tprev))
    np.testing.assert_allclose(ref.theta_vec(out["Tprev"]), th_k, rtol=0, atol=1e-13)
    np.testing.assert_allclose(ref.theta_vec(out["Tt"]), th_next, rtol=0, atol=1e-13)
    assert np.all(np.diag(out["Tprev"]) == 0) and np.all(np.diag(out["Tt"]) == 0)
    assert out["t"] == tn
    np.testing.assert_allclose(out["y"], y, atol=1e-12)
    np.testing.assert_allclose(out["xi"], xi, atol=1e-11)


# ---------------------------------------------------------------- P1 step from zero
def test_first_step_from_zero_closed_form():
    """P1: theta^0 = 0 => eta(0) = (ybar, 0), R_ij = ybar_j - ybar_i, Theta^1_ij = (ybar_i - ybar_j)_+ / L."""
    X, ybar = _tiny(9, 2, seed=7)
    L = 123.0
    out = oracle.papg(X, ybar, 1e-3, L, 1)
    want = np.maximum(0.0, ybar[:, None] - ybar[None, :]) / L
    np.fill_diagonal(want, 0.0)
    np.testing.assert_allclose(out["Tprev"], want, rtol=1e-15, atol=0)
    np.testing.assert_allclose(out["Tt"], want, rtol=1e-15, atol=0)  # beta_1 = (t_1-1)/t_2 = 0
    np.testing.assert_array_equal(out["y"], ybar)
    np.testing.assert_array_equal(out["xi"], 0.0)


# ---------------------------------------------------------------- P11 constant ybar
def test_constant_ybar_is_a_fixed_point():
    """P11: ybar constant => C eta(0) = 0 => Theta stays 0, y = ybar, xi = 0 for every k."""
    X, _ = _tiny(12, 3, seed=2)
    ybar = np.full(12, 2.5)
    out = oracle.papg(X, ybar, 1e-3, 50.0, 25)
    assert np.all(out["Tprev"] == 0) and np.all(out["Tt"] == 0)
    np.testing.assert_array_equal(out["y"], ybar)
    np.testing.assert_array_equal(out["xi"], 0.0)


# ---------------------------------------------------------------- P4 N=2 worked example
@pytest.mark.parametrize("case", [0, 1])
def test_n2_closed_form(case):
    """P4: N=2 closed form (tests/golden/n2_closed_form.json) -- NNLS and the oracle APG both reach it."""
    g = _gold("n2_closed_form.json")
    c = g["cases"][case]
    X, ybar, gamma = np.array(g["X"]), np.array(g["ybar"]), c["gamma"]
    opt = ref.regularized_optimum(X, ybar, gamma)
    np.testing.assert_allclose(opt["y"], c["y"], atol=1e-12)
    np.testing.assert_allclose(opt["xi"][:, 0], c["xi"], atol=1e-12)
    np.testing.assert_allclose(opt["theta"], [c["theta12"], c["theta21"]], atol=1e-12)
    L = ref.lipschitz(X, gamma)
    out = oracle.papg(X, ybar, gamma, L, 4000)
    y, xi = oracle.eta(X, ybar, gamma, out["Tprev"])
    np.testing.assert_allclose(y, c["y"], atol=1e-7)
    np.testing.assert_allclose(out["Tprev"][0, 1], c["theta12"], rtol=1e-6)
    assert out["Tprev"][1, 0] == 0.0


# ---------------------------------------------------------------- P3 / P5 / P6 / P7 / P13
@pytest.fixture(scope="module")
def small_run():
    N, n, gamma = 7, 2, 0.05
    X, ybar = _tiny(N, n, seed=11)
    L = ref.lipschitz(X, gamma)
    opt = ref.regularized_optimum(X, ybar, gamma)
    return dict(N=N, n=n, gamma=gamma, X=X, ybar=ybar, L=L, opt=opt)


def test_apg_reaches_nnls_optimum(small_run):
    """P3: oracle APG -> exact regularized optimum (Lawson-Hanson NNLS of the dual)."""
    s = small_run
    out = oracle.papg(s["X"], s["ybar"], s["gamma"], s["L"], 20000)
    y, xi = oracle.eta(s["X"], s["ybar"], s["gamma"], out["Tprev"])
    np.testing.assert_allclose(y, s["opt"]["y"], atol=1e-9)
    np.testing.assert_allclose(xi, s["opt"]["xi"], atol=1e-8)
    st = oracle.stats(s["X"], s["ybar"], s["gamma"], out["Tprev"], y, xi)
    # P7 KKT: primal objective equals p*, complementarity gap -> 0, violation -> 0
    assert abs(st["r_gamma"] - s["opt"]["p"]) <= 1e-10 * s["opt"]["p"]
    assert abs(st["gap"]) < 1e-9
    assert st["max_violation"] < 1e-8


def test_theorem1_envelope_and_apg_rate(small_run):
    """P5 Theorem 1 and P6 APG rate at every iterate; P13 invariants."""
    s = small_run
    X, ybar, gamma, L = s["X"], s["ybar"], s["gamma"], s["L"]
    p, ys, xis = s["opt"]["p"], s["opt"]["y"], s["opt"]["xi"]
    th_star = s["opt"]["theta"]
    R0 = float(th_star @ th_star)                      # ||theta^0 - theta*||^2 with theta^0 = 0
    N = s["N"]
    Tprev, Tt, t = np.zeros((N, N)), np.zeros((N, N)), 1.0
    for k in range(1, 301):
        out = oracle.papg(X, ybar, gamma, L, 1, Tprev=Tprev, Tt=Tt, t=t)
        Tprev, Tt, t_next = out["Tprev"], out["Tt"], out["t"]
        assert np.all(Tprev >= 0) and np.all(np.diag(Tprev) == 0)          # P13
        assert t_next >= (k + 2) / 2 - 1e-12                                 # t_{k+1} >= (k+2)/2
        g = ref.dual_value_dense(ref.theta_vec(Tprev), X, ybar, gamma)
        y, xi = oracle.eta(X, ybar, gamma, Tprev)
        lhs = np.sum((y - ys) ** 2) + gamma * np.sum((xi - xis) ** 2)
        assert lhs <= 2 * (p - g) + 1e-10                                   # Theorem 1
        assert p - g <= 2 * L * R0 / (k + 1) ** 2 + 1e-10                   # APG rate
        st = oracle.stats(X, ybar, gamma, Tprev, y, xi)
        assert abs(st["g"] - g) < 1e-10 * max(1.0, abs(g))                  # g = L(eta(theta), theta)
        t = t_next


def test_stats_against_dense(small_run):
    """oracle_stats vs dense C eta for a random (theta, eta)."""
    s = small_run
    X, ybar, gamma, N = s["X"], s["ybar"], s["gamma"], s["N"]
    rng = np.random.default_rng(5)
    T = crdata.random_theta(N, seed=3)
    y, xi = rng.standard_normal(N), rng.standard_normal((N, s["n"]))
    st = oracle.stats(X, ybar, gamma, T, y, xi)
    z = ref.dense_C(X) @ np.concatenate([y, xi.reshape(-1)])
    neg = np.minimum(z, 0)
    assert abs(st["gap"] - ref.theta_vec(T) @ z) < 1e-12
    assert abs(st["max_violation"] - max(0.0, -z.min())) < 1e-13
    assert abs(st["infeas_norm"] - np.linalg.norm(neg) / math.sqrt(N * N - N)) < 1e-13
    rg = 0.5 * np.sum((y - ybar) ** 2) + 0.5 * gamma * np.sum(xi ** 2)
    assert abs(st["r_gamma"] - rg) < 1e-12


# ---------------------------------------------------------------- P12 gradient
def test_gradient_is_minus_C_eta_finite_differences():
    """P12: grad g = -C eta(theta) (Eq. (dual gradient) P:370) vs central differences of g."""
    N, n, gamma = 5, 2, 0.1
    X, ybar = _tiny(N, n, seed=21)
    th = ref.theta_vec(crdata.random_theta(N, seed=22, density=1.0))
    grad = ref.dual_grad_dense(th, X, ybar, gamma)
    h = 1e-6
    for r in range(0, len(th), 3):
        e = np.zeros_like(th)
        e[r] = h
        fd = (ref.dual_value_dense(th + e, X, ybar, gamma) - ref.dual_value_dense(th - e, X, ybar, gamma)) / (2 * h)
        assert abs(fd - grad[r]) <= 1e-5 * max(1.0, abs(grad[r]))
    # the oracle's pair residual is the same C eta
    T = ref.theta_mat(th, N)
    y, xi = oracle.eta(X, ybar, gamma, T)
    st = oracle.stats(X, ybar, gamma, T, y, xi)
    assert abs(st["gap"] - th @ (-grad)) < 1e-10


# ---------------------------------------------------------------- P9 uniqueness of y*
def test_uniqueness_of_y_from_two_starts():
    """P9: N >= n+1 -- APG from theta^0 = 0 and from a random theta^0 >= 0 reach the same y."""
    N, n, gamma = 8, 2, 0.05
    X, ybar = _tiny(N, n, seed=31)
    L = ref.lipschitz(X, gamma)
    a = oracle.papg(X, ybar, gamma, L, 20000)
    T0 = crdata.random_theta(N, seed=32, scale=0.5)
    b = oracle.papg(X, ybar, gamma, L, 20000, Tprev=T0, Tt=T0)
    ya, _ = oracle.eta(X, ybar, gamma, a["Tprev"])
    yb, _ = oracle.eta(X, ybar, gamma, b["Tprev"])
    opt = ref.regularized_optimum(X, ybar, gamma)
    np.testing.assert_allclose(ya, yb, atol=1e-8)
    np.testing.assert_allclose(ya, opt["y"], atol=1e-8)


# ---------------------------------------------------------------- P8 univariate / Lemma 1
@pytest.mark.parametrize("gamma", [1e-2, 1e-4])
def test_univariate_lemma1_against_sorted_slope_fit(gamma):
    """P8: n=1, ||y*_gamma - y*|| <= ||xi*|| sqrt(gamma) (Lemma 1) with y* the 1-D convex LS fit.

    xi* (least-norm, Eq. (tikhonov)) is the projection of 0 onto each point's
    subdifferential interval [left slope, right slope] of the fitted interpolant.
    """
    N = 25
    rng = np.random.default_rng(41)
    x = np.sort(rng.uniform(-1, 1, N))
    ybar = x ** 2 + 0.1 * rng.standard_normal(N)
    ystar = ref.convex_fit_1d(x, ybar)
    slopes = np.diff(ystar) / np.diff(x)
    lo = np.concatenate([[-np.inf], slopes])
    hi = np.concatenate([slopes, [np.inf]])
    assert np.all(lo <= hi + 1e-9)                       # convex fit
    xi_star = np.clip(0.0, lo, hi)
    opt = ref.regularized_optimum(x[:, None], ybar, gamma)
    dist = np.linalg.norm(opt["y"] - ystar)
    assert dist <= np.linalg.norm(xi_star) * math.sqrt(gamma) * (1 + 1e-6) + 1e-9
    # the oracle APG approaches the same regularized optimum
    L = ref.lipschitz(x[:, None], gamma)
    out = oracle.papg(x[:, None], ybar, gamma, L, 3000 if gamma > 1e-3 else 8000)
    y, _ = oracle.eta(x[:, None], ybar, gamma, out["Tprev"])
    p = opt["p"]
    g = ref.dual_value_dense(ref.theta_vec(out["Tprev"]), x[:, None], ybar, gamma)
    assert np.sum((y - opt["y"]) ** 2) <= 2 * (p - g) + 1e-10   # Theorem 1 along the way


# ---------------------------------------------------------------- P10 L
@pytest.mark.parametrize("N", [3, 6, 20])
def test_lemma4_sigma_A1(N):
    """P10: sigma_max(A1)^2 = 2N (Lemma 4): with X = 0, C^T C = diag(A1^T A1, 0)."""
    X = np.zeros((N, 2))
    for form in ("definition", "structured"):
        assert abs(ref.sigma_max_sq(X, form) - 2 * N) < 1e-9 * N


@pytest.mark.parametrize("N,n,seed", [(4, 1, 0), (6, 2, 1), (8, 3, 2)])
def test_sigma_max_vs_dense_svd_and_bound(N, n, seed):
    """P10: Lanczos sigma_max(C) == dense SVD (N <= 8) and <= sqrt(2N) + B_x N (Lemma 4)."""
    X, _ = _tiny(N, n, seed)
    s_dense = np.linalg.svd(ref.dense_C(X), compute_uv=False)[0]
    for form in ("definition", "structured"):
        assert abs(math.sqrt(ref.sigma_max_sq(X, form)) - s_dense) < 1e-10 * s_dense
    Bx = np.linalg.norm(X, axis=1).max()
    assert s_dense <= math.sqrt(2 * N) + Bx * N


@pytest.mark.parametrize("N,n", [(9, 2), (40, 5), (130, 7)])
def test_structured_CtC_equals_definition(N, n):
    """The O(N n^2) C^T C product (derived) equals the pair-by-pair definition on random vectors."""
    X, _ = _tiny(N, n, seed=N)
    rng = np.random.default_rng(N)
    for _ in range(3):
        v = rng.standard_normal(N * (n + 1))
        a, b = ref.CtC_definition(X, v, chunk=17), ref.CtC_structured(X, v)
        np.testing.assert_allclose(b, a, rtol=0, atol=1e-10 * np.abs(a).max())
    if N <= 9:
        M = ref.dense_C(X)
        v = rng.standard_normal(N * (n + 1))
        np.testing.assert_allclose(ref.CtC_definition(X, v), M.T @ (M @ v), atol=1e-10)


def test_lipschitz_bounds_gradient_variation():
    """L_gamma (Eq. (lischitz), gamma <= 1) bounds ||grad g(a) - grad g(b)|| / ||a - b||."""
    N, n, gamma = 6, 2, 0.2
    X, ybar = _tiny(N, n, seed=51)
    L = ref.lipschitz(X, gamma)
    rng = np.random.default_rng(52)
    for _ in range(10):
        a, b = rng.exponential(size=N * (N - 1)), rng.exponential(size=N * (N - 1))
        ga, gb = ref.dual_grad_dense(a, X, ybar, gamma), ref.dual_grad_dense(b, X, ybar, gamma)
        assert np.linalg.norm(ga - gb) <= L * np.linalg.norm(a - b) * (1 + 1e-12)


# ---------------------------------------------------------------- determinism / threads
def test_oracle_independent_of_thread_count():
    X, ybar = _tiny(300, 3, seed=61)
    a = oracle.papg(X, ybar, 1e-3, 500.0, 3, nthreads=1)
    b = oracle.papg(X, ybar, 1e-3, 500.0, 3, nthreads=4)
    np.testing.assert_array_equal(a["Tt"], b["Tt"])
    np.testing.assert_array_equal(a["xi"], b["xi"])


def test_project_rows_matches_full_step():
    """oracle_project_rows (sampled Step 2) == rows of a full oracle step."""
    X, ybar = _tiny(50, 3, seed=71)
    T = crdata.random_theta(50, seed=72, scale=1e-3)
    out = oracle.papg(X, ybar, 1e-3, 900.0, 1, Tprev=T, Tt=T)
    rows = np.array([0, 7, 49])
    got = oracle.project_rows(X, out["y"], out["xi"], 900.0, rows, T[rows])
    np.testing.assert_array_equal(got, out["Tprev"][rows])


def test_config_generators_are_seeded_and_fp32_rounded():
    X1, y1 = crdata.make_problem("C2", N=200)
    X2, y2 = crdata.make_problem("C2", N=200)
    np.testing.assert_array_equal(X1, X2)
    assert np.all(X1.astype(np.float32).astype(np.float64) == X1)
    Xc, yc = crdata.make_problem("C1")
    assert Xc.shape == (50, 2) and np.abs(Xc).max() <= 1


# ---------------------------------------------------------------- adaptive step
def _adaptive_check_dense(theta_t, theta_k, s, X, ybar, gamma):
    """Eq. (adaptive-check) evaluated with the dense Def. A1A2 operators:
    g(theta^k) - [g(theta~) + <grad g(theta~), theta^k - theta~> - s/2 ||theta^k - theta~||^2]."""
    tt, tk = ref.theta_vec(theta_t), ref.theta_vec(theta_k)
    D = tk - tt
    lhs = ref.dual_value_dense(tk, X, ybar, gamma)
    rhs = ref.dual_value_dense(tt, X, ybar, gamma) + ref.dual_grad_dense(tt, X, ybar, gamma) @ D - 0.5 * s * (D @ D)
    return lhs - rhs


def _dense_step(theta_t, s, X, ybar, gamma):
    """Step 2 with step 1/s: (theta~ - C eta(theta~) / s)_+, dense."""
    tt = ref.theta_vec(theta_t)
    return ref.theta_mat(np.maximum(tt + ref.dual_grad_dense(tt, X, ybar, gamma) / s, 0.0), X.shape[0])


@pytest.mark.parametrize("N,n,seed,ups", [(6, 2, 0, 2.0), (8, 3, 1, 2.0), (7, 1, 2, 3.0)])
def test_adaptive_rule_accepts_minimal_l(N, n, seed, ups):
    """PAPG_A: every accepted s_k = s_{k-1} ups^(l_k - 1) satisfies Eq. (adaptive-check)
    and l_k is minimal (the trial at s_k / ups fails), both re-evaluated with dense operators."""
    X, ybar = _tiny(N, n, seed)
    gamma = 0.05
    L = ref.lipschitz(X, gamma)
    st = dict(Tprev=None, Tt=None, t=1.0, s=L)
    for k in range(25):
        Tt = np.zeros((N, N)) if st["Tt"] is None else st["Tt"]
        nxt = oracle.papg_adaptive(X, ybar, gamma, st["s"], 1, ups=ups, Tprev=st["Tprev"], Tt=st["Tt"], t=st["t"])
        s_k, l_k = nxt["s_hist"][0], int(nxt["trials"][0]) - 1
        assert math.isclose(s_k, st["s"] * ups ** (l_k - 1), rel_tol=1e-15)
        Tk = nxt["Tprev"]
        np.testing.assert_allclose(Tk, _dense_step(Tt, s_k, X, ybar, gamma), rtol=1e-10, atol=1e-14)
        scale = 1.0 + abs(ref.dual_value_dense(ref.theta_vec(Tt), X, ybar, gamma))
        assert _adaptive_check_dense(Tt, Tk, s_k, X, ybar, gamma) >= -1e-12 * scale
        if l_k >= 1:
            Tr = _dense_step(Tt, s_k / ups, X, ybar, gamma)
            assert _adaptive_check_dense(Tt, Tr, s_k / ups, X, ybar, gamma) < 0
        st = dict(Tprev=nxt["Tprev"], Tt=nxt["Tt"], t=nxt["t"], s=nxt["s"])


def test_adaptive_with_huge_ups_is_constant_step():
    """With ups = 1e30 the l = 0 trial (step 1e30/s) always fails and l = 1 (s_k = s_{k-1} = L)
    always passes (descent lemma: L bounds the gradient's Lipschitz constant, Eq. (lischitz)
    P:375), so PAPG_A reproduces the constant-step Fig. 2 iterates with 2 trials per iteration."""
    X, ybar = _tiny(12, 2, seed=4)
    gamma = 0.02
    L = ref.lipschitz(X, gamma)
    a = oracle.papg_adaptive(X, ybar, gamma, L, 30, ups=1e30)
    c = oracle.papg(X, ybar, gamma, L, 30)
    assert np.all(a["trials"] == 2)
    assert np.all(a["s_hist"] == L)
    np.testing.assert_allclose(a["Tprev"], c["Tprev"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(a["y"], c["y"], rtol=0, atol=1e-13)


def test_adaptive_quadratic_identity():
    """g is quadratic at K = N (Step 1 is unconstrained), so for any theta, D:
    g(theta+D) - g(theta) - <grad g(theta), D> = -1/2 (||A1^T D||^2 + ||A2^T D||^2 / gamma).
    This is the form the GPU evaluates Eq. (adaptive-check) in (reading R15)."""
    X, ybar = _tiny(7, 2, seed=5)
    gamma = 0.03
    rng = np.random.default_rng(0)
    M = 7 * 6
    for _ in range(5):
        th, D = rng.random(M), rng.standard_normal(M)
        lhs = (ref.dual_value_dense(th + D, X, ybar, gamma) - ref.dual_value_dense(th, X, ybar, gamma)
               - ref.dual_grad_dense(th, X, ybar, gamma) @ D)
        A1D, A2D = ref.dense_A1(7).T @ D, ref.dense_A2(X).T @ D
        assert math.isclose(lhs, -0.5 * (A1D @ A1D + A2D @ A2D / gamma), rel_tol=1e-9)


def test_adaptive_converges_to_nnls_optimum_within_backtracking_rate():
    """PAPG_A reaches the exact regularized optimum (P3) and obeys the backtracking-APG rate
    p* - g(theta^k) <= 2 max_k(s_k) ||theta^0 - theta*||^2 / (k+1)^2 (P:341 with L -> max s_k)."""
    X, ybar = _tiny(8, 2, seed=6)
    gamma = 0.05
    opt = ref.regularized_optimum(X, ybar, gamma)
    L = ref.lipschitz(X, gamma)
    st = dict(Tprev=None, Tt=None, t=1.0, s=L)
    smax = 0.0
    th2 = opt["theta"] @ opt["theta"]
    for k in range(1, 401):
        nxt = oracle.papg_adaptive(X, ybar, gamma, st["s"], 1, Tprev=st["Tprev"], Tt=st["Tt"], t=st["t"])
        smax = max(smax, nxt["s_hist"][0])
        g = ref.dual_value_dense(ref.theta_vec(nxt["Tprev"]), X, ybar, gamma)
        assert opt["p"] - g <= 2 * smax * th2 / (k + 1) ** 2 + 1e-10
        st = dict(Tprev=nxt["Tprev"], Tt=nxt["Tt"], t=nxt["t"], s=nxt["s"])
    y, _ = oracle.eta(X, ybar, gamma, st["Tprev"])
    # (near the optimum the literal check's rounding -- g values of O(||ybar||^2) differenced to
    # O(||D||^2) -- rejects steps spuriously and s_k grows; 400 iterations stay clear of that)
    np.testing.assert_allclose(y, opt["y"], atol=5e-6)


# ---------------------------------------------------------------- continuation (Section 2.4.1)
def test_continuation_approaches_unregularized_estimator_1d():
    """Continuation on a univariate problem: as gamma_t = kappa eps0 / beta^t -> 0 the
    stage estimators y^(t) approach the exact unregularized convex LS fit y* (sorted-slope fit, a
    textbook routine) within ||xi*|| sqrt(gamma_t) + sqrt(2 delta_t), delta_t the dual
    suboptimality of stage t measured against the exact regularized optimum (NNLS, P3)."""
    N = 20
    rng = np.random.default_rng(7)
    x = np.sort(rng.uniform(-1, 1, N))
    ybar = x ** 2 + 0.1 * rng.standard_normal(N)
    X = x[:, None]
    ystar = ref.convex_fit_1d(x, ybar)
    slopes = np.diff(ystar) / np.diff(x)
    xi_star = np.clip(0.0, np.concatenate([[-np.inf], slopes]), np.concatenate([slopes, [np.inf]]))
    sigma2 = ref.sigma_max_sq(X)
    stages = oracle.continuation(X, ybar, sigma2, eps0=1e-1, beta=4.0, kappa_gamma=1.0, iters=[3000] * 5)
    prev = np.inf
    for st in stages:
        opt = ref.regularized_optimum(X, ybar, st["gamma"])
        delta = opt["p"] - ref.dual_value_dense(ref.theta_vec(st["Theta"]), X, ybar, st["gamma"])
        assert delta >= -1e-10
        dist = np.linalg.norm(st["y"] - ystar)
        bound = np.linalg.norm(xi_star) * math.sqrt(st["gamma"]) + math.sqrt(2 * max(delta, 0.0))
        assert dist <= bound * (1 + 1e-6) + 1e-9, (st["gamma"], dist, bound)
        prev = min(prev, dist)
    assert np.linalg.norm(stages[-1]["y"] - ystar) < np.linalg.norm(stages[0]["y"] - ystar)


def test_continuation_stage_is_warm_started_papg():
    """Stage t is Fig. 2 restarted at theta^(t-1) (theta~^1 = theta^0, t_1 = 1) with
    L_t = sigma_max(C)^2 / gamma_t (Eq. (lischitz)): a 1-stage continuation from Theta0
    equals oracle.papg from (Theta0, Theta0, 1) -- and its first step from 0 is Theta^1 of P1."""
    X, ybar = _tiny(10, 2, seed=8)
    sigma2 = ref.sigma_max_sq(X)
    st = oracle.continuation(X, ybar, sigma2, eps0=0.5, beta=2.0, kappa_gamma=0.1, iters=[1])[0]
    assert math.isclose(st["gamma"], 0.1 * 0.5 / 2.0)
    want = np.maximum(ybar[:, None] - ybar[None, :], 0.0) / (sigma2 / st["gamma"])
    np.fill_diagonal(want, 0.0)
    np.testing.assert_allclose(st["Theta"], want, rtol=1e-14, atol=0)
    T0 = crdata.random_theta(10, seed=3)
    a = oracle.continuation(X, ybar, sigma2, eps0=0.5, beta=2.0, kappa_gamma=0.1, iters=[7, 5], Theta0=T0)
    b1 = oracle.papg(X, ybar, a[0]["gamma"], a[0]["L"], 7, Tprev=T0, Tt=T0, t=1.0)
    b2 = oracle.papg(X, ybar, a[1]["gamma"], a[1]["L"], 5, Tprev=b1["Tprev"], Tt=b1["Tprev"], t=1.0)
    np.testing.assert_array_equal(a[1]["Theta"], b2["Tprev"])


def test_continuation_stop_branch_is_the_p1106_pair_at_multiples_of_m():
    """The early stop inside a continuation stage (oracle/core.py, the ``stop`` branch): with
    stop = (m, infeas_tol, gap_tol) a stage ends at the FIRST multiple k of m at which the stopping
    pair of P:1106 holds at eta(theta^k) -- normalized infeasibility ||(C eta)_-|| / sqrt(N^2 - N)
    <= infeas_tol and |theta^T C eta| / (N^2 - N) <= gap_tol -- and returns theta^k of Fig. 2.
    Both conditions are re-evaluated here with the dense operators of Def. A1A2, so
    the pin is independent of oracle_eta / oracle_stats."""
    N, n, m = 8, 2, 5
    X, ybar = _tiny(N, n, seed=31)
    sigma2 = ref.sigma_max_sq(X)
    eps0, beta, kap = 0.5, 2.0, 0.02
    gamma = kap * eps0 / beta
    L = sigma2 / gamma
    C = ref.dense_C(X)
    # the dense stopping quantities at theta^k for k = m, 2m, ...
    hist = []
    st = dict(Tprev=np.zeros((N, N)), Tt=np.zeros((N, N)), t=1.0)
    for k in range(m, 401, m):
        st = oracle.papg(X, ybar, gamma, L, m, Tprev=st["Tprev"], Tt=st["Tt"], t=st["t"])
        th = ref.theta_vec(st["Tprev"])
        y, xi = ref.eta_dense(th, X, ybar, gamma)
        z = C @ np.concatenate([y, xi.reshape(-1)])
        hist.append((k, np.linalg.norm(np.minimum(z, 0.0)) / math.sqrt(N * N - N), abs(th @ z) / (N * N - N),
                     st["Tprev"].copy()))
    # tolerances placed between consecutive checks, so exactly one k is the first to satisfy both
    inf_tol = 0.5 * (hist[5][1] + hist[6][1]) if hist[6][1] < hist[5][1] else hist[6][1] * (1 + 1e-9)
    gap_tol = max(h[2] for h in hist) * 2 + 1e-300
    first = next(h for h in hist if h[1] <= inf_tol and h[2] <= gap_tol)
    assert m < first[0] < 400
    st = oracle.continuation(X, ybar, sigma2, eps0=eps0, beta=beta, kappa_gamma=kap, iters=[400],
                             stop=(m, inf_tol, gap_tol))[0]
    assert st["iters"] == first[0]
    np.testing.assert_array_equal(st["Theta"], first[3])
    # a gap tolerance no iterate meets: the stage runs its whole budget
    st2 = oracle.continuation(X, ybar, sigma2, eps0=eps0, beta=beta, kappa_gamma=kap, iters=[40],
                              stop=(m, inf_tol, -1.0))[0]
    assert st2["iters"] == 40
    np.testing.assert_array_equal(st2["Theta"], hist[7][3])


# ---------------------------------------------------------------- max-affine estimator
def test_predict_from_exact_convex_supports():
    """With y_i = f(x_i), xi_i = grad f(x_i) of a convex f (every pair constraint of Eq. (original)
    P:64 holds by the gradient inequality), f_hat interpolates f at the data points and lies
    below f everywhere (it is a max of supporting hyperplanes)."""
    rng = np.random.default_rng(0)
    X = rng.standard_normal((40, 3))
    A = rng.standard_normal((3, 3))
    Q = A @ A.T + 0.1 * np.eye(3)
    f = lambda Z: 0.5 * np.einsum("ij,jk,ik->i", Z, Q, Z)
    y, xi = f(X), X @ Q
    np.testing.assert_allclose(ref.predict(X, y, xi, X), y, rtol=0, atol=1e-12)
    Z = rng.standard_normal((200, 3)) * 2
    assert np.all(ref.predict(X, y, xi, Z) <= f(Z) + 1e-12)
    # a single data point: f_hat is that point's supporting hyperplane
    z = rng.standard_normal((5, 3))
    np.testing.assert_allclose(ref.predict(X[:1], y[:1], xi[:1], z), y[0] + (z - X[0]) @ xi[0], rtol=1e-14)


def test_backtrack_variant_monotone_minimal_and_constant_from_L():
    """The monotone variant (R18): s_k = s_{k-1} ups^(l_k), so accepted s_k never decrease;
    each accepted step passes Eq. (adaptive-check) (dense re-evaluation) and l_k is minimal; started
    at s_0 = L it is the constant-step Fig. 2 (L bounds the gradient's Lipschitz constant)."""
    X, ybar = _tiny(8, 2, seed=9)
    gamma = 0.05
    L = ref.lipschitz(X, gamma)
    st = dict(Tprev=None, Tt=None, t=1.0, s=L / 64)
    prev_s = 0.0
    for k in range(20):
        Tt = np.zeros((8, 8)) if st["Tt"] is None else st["Tt"]
        nxt = oracle.papg_adaptive(X, ybar, gamma, st["s"], 1, Tprev=st["Tprev"], Tt=st["Tt"], t=st["t"],
                                   backtrack=True)
        s_k, l_k = nxt["s_hist"][0], int(nxt["trials"][0]) - 1
        assert s_k >= prev_s and math.isclose(s_k, st["s"] * 2.0 ** l_k, rel_tol=1e-15)
        Tk = nxt["Tprev"]
        scale = 1.0 + abs(ref.dual_value_dense(ref.theta_vec(Tt), X, ybar, gamma))
        assert _adaptive_check_dense(Tt, Tk, s_k, X, ybar, gamma) >= -1e-12 * scale
        if l_k >= 1:
            Tr = _dense_step(Tt, s_k / 2.0, X, ybar, gamma)
            assert _adaptive_check_dense(Tt, Tr, s_k / 2.0, X, ybar, gamma) < 0
        prev_s = s_k
        st = dict(Tprev=nxt["Tprev"], Tt=nxt["Tt"], t=nxt["t"], s=nxt["s"])
    a = oracle.papg_adaptive(X, ybar, gamma, L, 25, backtrack=True)
    c = oracle.papg(X, ybar, gamma, L, 25)
    assert np.all(a["trials"] == 1) and np.all(a["s_hist"] == L)
    np.testing.assert_array_equal(a["Tprev"], c["Tprev"])


def test_paper_section4_generator():
    """crdata.paper_problem follows P:943-944 (reading R19): cond(Q) = 15, x ~ N(0, 4), 30% of the
    points moved to 1.3 ybar; seeded (same seed, same data)."""
    import crdata as cd
    X, y = cd.paper_problem(3000, 6, "quad", seed=3)
    X2, y2 = cd.paper_problem(3000, 6, "quad", seed=3)
    np.testing.assert_array_equal(X, X2)
    np.testing.assert_array_equal(y, y2)
    assert abs(X.var() - 4.0) < 0.1
    rng = np.random.default_rng(3)
    Xr = 2.0 * rng.standard_normal(size=(3000, 6))
    np.testing.assert_array_equal(X, Xr)                      # X is drawn first
    Lam = rng.standard_normal(size=(6, 6))
    sv = np.linalg.svd(Lam.T @ Lam, compute_uv=False)
    assert sv.max() / sv.min() > 15                          # the transform is needed
    Xe, ye = cd.paper_problem(2000, 4, "exp", seed=1)
    rng = np.random.default_rng(1)
    Xr = 2.0 * rng.standard_normal(size=(2000, 4))
    p = rng.uniform(0.0, 0.2, size=4)
    f = np.exp(Xr @ p)
    eps = 10.0 * rng.standard_normal(size=2000)
    moved = rng.choice(2000, size=600, replace=False)
    want = f + eps
    want[moved] *= 1.3
    np.testing.assert_allclose(ye, want, rtol=1e-15)


# ---------------------------------------------------------------- general partition K < N (Section 2.1)
def test_partition_nbar1_is_the_all_pairs_method():
    """Nbar = 1 (K = N singleton blocks): no intra-block constraints, Step 1 is the closed form."""
    from oracle import partition
    X, ybar = _tiny(12, 2, seed=61)
    L = ref.lipschitz(X, 0.05)
    a = partition.papg_partition(X, ybar, 0.05, L, 30, 1)
    b = oracle.papg(X, ybar, 0.05, L, 30)
    np.testing.assert_allclose(a["Tprev"], b["Tprev"], rtol=0, atol=1e-14)
    np.testing.assert_allclose(a["y"], b["y"], rtol=0, atol=1e-12)


def test_partition_single_block_solves_the_qp_in_step1():
    """Nbar = N (K = 1): nothing is dualized and Step 1 at theta = 0 is the regularized QP itself,
    so eta^1 is the exact regularized optimum (P3, NNLS) and Theta stays 0."""
    from oracle import partition
    X, ybar = _tiny(7, 2, seed=62)
    gamma = 0.05
    opt = ref.regularized_optimum(X, ybar, gamma)
    a = partition.papg_partition(X, ybar, gamma, ref.lipschitz(X, gamma), 1, 7)
    np.testing.assert_allclose(a["y"], opt["y"], atol=1e-9)
    np.testing.assert_allclose(a["xi"], opt["xi"], atol=1e-8)
    assert np.all(a["Tprev"] == 0)


def test_block_projection_kkt():
    """The block projection satisfies its KKT conditions: feasibility, lambda >= 0, stationarity
    (by construction), complementarity lambda_p (A eta)_p = 0."""
    from oracle import partition
    rng = np.random.default_rng(63)
    Xb = rng.standard_normal((6, 2))
    y0, xi0 = rng.standard_normal(6), rng.standard_normal((6, 2))
    y, xi, lam = partition.project_block(Xb, y0, xi0, 0.1)
    Ae = ref.dense_A1(6) @ y + ref.dense_A2(Xb) @ xi.reshape(-1)
    assert Ae.min() >= -1e-9 and lam.min() >= 0
    assert abs(lam @ Ae) <= 1e-8 * (1 + np.abs(lam).sum())


def test_partition_converges_to_regularized_optimum():
    """Any partition solves the same dual problem's primal (strong duality): P-APG with
    Nbar = 4 on N = 12 reaches the exact regularized optimum (P3)."""
    from oracle import partition
    X, ybar = _tiny(12, 2, seed=64)
    gamma = 0.05
    opt = ref.regularized_optimum(X, ybar, gamma)
    L = ref.lipschitz(X, gamma)
    a = partition.papg_partition(X, ybar, gamma, L, 3000, 4)
    y, xi = partition.eta_partition(X, ybar, gamma, a["Tprev"], 4)
    np.testing.assert_allclose(y, opt["y"], atol=3e-5)      # 8e-6 at 3000 iterations (all-pairs: 3e-6)
