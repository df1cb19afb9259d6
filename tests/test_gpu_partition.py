"""GPU parity for the general partition K < N (Assumption 1, R20):
libcr with cr_config.nbar = Nbar vs oracle/partition.py on the same seeded inputs.

Only cross-block pairs carry a dual variable; Step 1 is the closed-form point projected per
block onto the intra-block constraints (Eq. (subgradient_split)).  The oracle solves
each projection exactly through its NNLS dual; libcr by an fp64 interior-point kernel (to a
relative 1e-9) followed by an exact active-set polish (R20), so fp64 runs agree to
~1e-12 per projection (1e-8 asserted on Theta after several iterations, whose small entries
amplify the error) and fp32 runs to the fp32 bar of the K = N tests.
"""
import threading

import numpy as np
import pytest

import crdata
import oracle
from oracle import partition, ref

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def r32(a):
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


@pytest.mark.parametrize("N,n,nbar,K,gamma,seed", [
    (120, 3, 12, 8, 1e-2, 0),
    (96, 5, 32, 5, 1e-2, 1),
    (200, 2, 8, 10, 1e-3, 2),
    (400, 2, 100, 3, 1e-3, 3),               # the paper's block size
    (60, 1, 2, 6, 1e-2, 4),                  # smallest blocks (2 constraints each), n = 1
    (64, 7, 64, 3, 1e-2, 5),                 # one block of 64: Nbar = N, Theta = 0
])
def test_partition_iterations_fp64(crp, N, n, nbar, K, gamma, seed):
    X, ybar = crdata.random_problem(N, n, seed=seed)
    L = ref.lipschitz(X, gamma)
    want = partition.papg_partition(X, ybar, gamma, L, K, nbar)
    s = crp.Solver(X, ybar, gamma, L=L, prec="fp64", nbar=nbar)
    for _ in range(K):
        s.step()
    info = s.partition_info()
    assert info["nbar"] == nbar and info["ipm_iters_max"] < 100
    assert info["failed_blocks"] == 0 and info["unpolished_blocks"] == 0
    assert info["blocks"] == N // nbar and 0 < info["warm_blocks"] <= info["blocks"]     # warm starts in use
    T, _, tk, _ = s.get_theta()
    y, xi = s.get_eta()                      # eta of the last Step 1 (at theta~^K)
    mask = partition.block_mask(N, nbar)
    assert np.all(T[~mask] == 0) and np.all(T >= 0)
    assert rel(T, want["Tprev"]) <= 1e-8
    assert rel(y, want["y"]) <= 1e-9 and rel(xi, want["xi"]) <= 1e-8
    # eta(Theta^K) and the diagnostics (g = r_gamma - gap at K < N)
    yp, xip, st = s.primal()
    yw, xiw = partition.eta_partition(X, ybar, gamma, want["Tprev"], nbar)
    sw = oracle.stats(X, ybar, gamma, want["Tprev"], yw, xiw)
    assert rel(yp, yw) <= 1e-8 and rel(xip, xiw) <= 1e-8
    for k in ("r_gamma", "gap", "g"):
        assert abs(st[k] - sw[k]) <= 1e-7 * (abs(sw[k]) + abs(sw["r_gamma"])), (k, st[k], sw[k])
    s.close()


@pytest.mark.parametrize("N,n,nbar,kernel,K0,seed", [
    (300, 5, 20, "simt", 12, 3),
    (256, 16, 16, "tc", 10, 4),
    (384, 20, 48, "tc", 6, 5),               # blocks straddling the 32-column tiles
])
def test_partition_single_step_fp32(crp, N, n, nbar, kernel, K0, seed):
    """A mid-run oracle state (fp32-rounded) -> one GPU step vs one oracle step."""
    X, ybar = crdata.random_problem(N, n, seed=seed, fp32=True)
    gamma = 1e-3
    L = ref.lipschitz(X, gamma)
    st = partition.papg_partition(X, ybar, gamma, L, K0, nbar)
    # Theta^{K0-1} is not returned: rebuild the pair from K0-1 and K0 runs
    st1 = partition.papg_partition(X, ybar, gamma, L, K0 - 1, nbar)
    Tk, Tkm1 = r32(st["Tprev"]), r32(st1["Tprev"])
    t_k, t_kp1 = st1["t"], st["t"]
    Tt = oracle.extrapolate(Tk, Tkm1, t_k, t_kp1)
    want = partition.papg_partition(X, ybar, gamma, L, 1, nbar, Tprev=Tk, Tt=Tt, t=t_kp1)
    s = crp.Solver(X, ybar, gamma, L=L, prec="fp32", kernel=kernel, nbar=nbar)
    s.set_theta(Tk, Tkm1, t_k, t_kp1)
    s.step()
    T = s.get_theta()[0]
    y, xi = s.get_eta()
    assert np.all(T[~partition.block_mask(N, nbar)] == 0)
    assert rel(T, want["Tprev"]) <= 1e-5
    assert rel(y, want["y"]) <= 1e-5 and rel(xi, want["xi"]) <= 1e-5
    s.close()


def test_partition_cold_start_matches(crp, monkeypatch):
    """CR_IPM_COLD=1 (every projection by the interior point + polish) gives the same iterates."""
    N, n, nbar, K, gamma = 120, 3, 12, 6, 1e-2
    X, ybar = crdata.random_problem(N, n, seed=11)
    L = ref.lipschitz(X, gamma)
    want = partition.papg_partition(X, ybar, gamma, L, K, nbar)
    monkeypatch.setenv("CR_IPM_COLD", "1")
    s = crp.Solver(X, ybar, gamma, L=L, prec="fp64", nbar=nbar)
    s.solve(K)
    info = s.partition_info()
    assert info["warm_blocks"] == 0 and info["ipm_iters_max"] > 0
    assert rel(s.get_theta()[0], want["Tprev"]) <= 1e-8
    s.close()


def test_partition_single_block_solves_qp(crp):
    """Nbar = N (K = 1): no dual variables; Step 1 is the QP itself (P:184-187 with one block)."""
    N, n, gamma = 60, 2, 1e-2
    X, ybar = crdata.random_problem(N, n, seed=7)
    s = crp.Solver(X, ybar, gamma, L=1.0, prec="fp64", nbar=N)
    s.step()
    T = s.get_theta()[0]
    assert np.all(T == 0)
    y, xi, st = s.primal()
    yw, xiw = partition.eta_partition(X, ybar, gamma, np.zeros((N, N)), N)
    assert rel(y, yw) <= 1e-9 and rel(xi, xiw) <= 1e-8
    assert st["max_violation"] <= 1e-9 * np.abs(y).max()
    s.close()


def test_partition_nbar1_is_all_pairs(crp):
    """nbar = 1 is the K = N method bit for bit."""
    N, n, gamma, K = 150, 4, 1e-3, 6
    X, ybar = crdata.random_problem(N, n, seed=8, fp32=True)
    out = []
    for nb in (0, 1):
        s = crp.Solver(X, ybar, gamma, L=ref.lipschitz(X, gamma), prec="fp32", nbar=nb)
        s.solve(K)
        out.append(s.get_theta()[0])
        s.close()
    np.testing.assert_array_equal(out[0], out[1])


def test_partition_rejects(crp):
    X, ybar = crdata.random_problem(120, 3, seed=9)
    with pytest.raises(crp.CrError):
        crp.Solver(X, ybar, 1e-2, L=1.0, nbar=7)               # N % nbar != 0
    X2, y2 = crdata.random_problem(258, 3, seed=9)
    with pytest.raises(crp.CrError):
        crp.Solver(X2, y2, 1e-2, L=1.0, nbar=129)              # > 128
    with pytest.raises(crp.CrError):
        crp.Solver(X, ybar, 1e-2, L=1.0, nbar=12, adaptive=True)
    s = crp.Solver(X, ybar, 1e-2, L=1.0, prec="fp64", nbar=12)
    T = np.zeros((120, 120))
    T[0, 5] = 1.0                                               # intra-block pair (block 0)
    with pytest.raises(crp.CrError):
        s.set_theta(T, T)
    T[0, 5], T[0, 50] = 0.0, 1.0                                # cross-block: fine
    s.set_theta(T, T)
    s.close()


def test_partition_sharded_local_group(crp):
    """Row shards aligned to the blocks (S % nbar == 0), world 2 in one process."""
    import torch
    N, n, nbar, K, gamma = 240, 3, 12, 6, 1e-2
    X, ybar = crdata.random_problem(N, n, seed=10)
    L = ref.lipschitz(X, gamma)
    want = partition.papg_partition(X, ybar, gamma, L, K, nbar)
    g = crp.LocalGroup(2)
    res, errs = [None, None], []

    def body(r):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                sol = crp.Solver(X, ybar, gamma, L=L, prec="fp64", group=g, rank=r, stream=st, nbar=nbar)
                sol.solve(K)
                res[r] = dict(row0=sol.row0, T=sol.get_theta()[0], eta=sol.get_eta())
                sol.close()
            st.synchronize()
        except Exception as e:                                  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=body, args=(r,)) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    g.close()
    if errs:
        raise errs[0]
    T = np.zeros((N, N))
    xi = np.zeros((N, n))
    for r in res:
        T[r["row0"]:r["row0"] + r["T"].shape[0]] = r["T"]
        xi[r["row0"]:r["row0"] + r["eta"][1].shape[0]] = r["eta"][1]
    assert rel(T, want["Tprev"]) <= 1e-8
    assert rel(res[0]["eta"][0], want["y"]) <= 1e-9 and rel(xi, want["xi"]) <= 1e-8
