"""The row-sharded multi-GPU path of libcr run end to end on ONE GPU.

world > 1 contexts join an in-process local group (cr_local_group_create): each rank is a
Solver driven by its own host thread and CUDA stream, owning rows [r S, min(N, (r+1) S)),
S = ceil(N / world), exactly as under NCCL; the all-gather of y', the reduce-scatter of the
column sums and the scalar all-reduces are performed by the group (host rendezvous + event
dependencies + copies / a fixed-order sum kernel; no kernel waits on another).  The
assembled sharded iterates must match the fp64 oracle like the single-GPU path does.
"""
import threading

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


def run_ranks(crp, world, fn):
    """fn(rank, group, stream) on `world` threads; returns the per-rank results."""
    import torch
    g = crp.LocalGroup(world)
    out, errs = [None] * world, []

    def body(r):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                out[r] = fn(r, g, s)
            s.synchronize()
        except Exception as e:                      # noqa: BLE001
            errs.append((r, e))

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    g.close()
    if errs:
        raise errs[0][1]
    return out


@pytest.mark.parametrize("N,n,prec,kernel,world,K,tol", [
    (300, 5, "fp64", "auto", 2, 30, 1e-11),
    (301, 4, "fp64", "auto", 3, 25, 1e-11),       # ragged shards (101, 101, 99 rows)
    (1000, 20, "fp32", "tc", 2, 30, 2e-5),
    (517, 33, "fp32", "tc", 3, 20, 2e-5),         # ragged shards, partial 128-row blocks
    (900, 10, "fp32", "simt", 4, 20, 2e-5),
    (4000, 20, "fp32", "tc", 4, 20, 2e-5),        # C3 laws' size on 4 ranks (1000 rows each)
])
def test_sharded_solve_matches_oracle(crp, N, n, prec, kernel, world, K, tol):
    X, ybar = crdata.random_problem(N, n, seed=N + world, fp32=prec == "fp32")
    gamma = 1e-3
    L = ref.lipschitz(X, gamma)
    want = oracle.papg(X, ybar, gamma, L, K)
    yw, xiw = oracle.eta(X, ybar, gamma, want["Tprev"])
    sw = oracle.stats(X, ybar, gamma, want["Tprev"], yw, xiw)

    def fn(r, g, s):
        sol = crp.Solver(X, ybar, gamma, L=L, prec=prec, kernel=kernel, group=g, rank=r, stream=s)
        sol.solve(K)
        T = sol.get_theta()[0]
        y, xi, st = sol.primal()
        res = dict(row0=sol.row0, T=T, y=y, xi=xi, st=st)
        sol.close()
        return res

    res = run_ranks(crp, world, fn)
    T = np.zeros((N, N))
    xi = np.zeros((N, n))
    for r in res:
        T[r["row0"]:r["row0"] + r["T"].shape[0]] = r["T"]
        xi[r["row0"]:r["row0"] + r["xi"].shape[0]] = r["xi"]
        np.testing.assert_array_equal(r["y"], res[0]["y"])          # every rank holds the full y
        assert r["st"]["r_gamma"] == res[0]["st"]["r_gamma"]        # all-reduced diagnostics agree
    assert sum(r["T"].shape[0] for r in res) == N
    assert rel(T, want["Tprev"]) <= tol
    assert rel(res[0]["y"], yw) <= tol and rel(xi, xiw) <= tol
    st = res[0]["st"]
    assert abs(st["r_gamma"] - sw["r_gamma"]) <= 1e-4 * abs(sw["r_gamma"])
    assert abs(st["max_violation"] - sw["max_violation"]) <= 1e-4 * abs(sw["max_violation"]) + 1e-12


def test_sharded_single_step_from_state(crp):
    """cr_set_theta with each rank's own rows of a mid-run oracle state, then one step."""
    N, n, world = 600, 24, 2
    X, ybar = crdata.random_problem(N, n, seed=5, fp32=True)
    gamma = 1e-3
    L = ref.lipschitz(X, gamma)
    st = oracle.state_after(X, ybar, gamma, L, 15)
    r32 = lambda a: a.astype(np.float32).astype(np.float64)
    Tk, Tkm1 = r32(st["Tk"]), r32(st["Tkm1"])
    want = oracle.papg(X, ybar, gamma, L, 1, Tprev=Tk, Tt=oracle.extrapolate(Tk, Tkm1, st["t_k"], st["t_kp1"]),
                       t=st["t_kp1"])

    def fn(r, g, s):
        sol = crp.Solver(X, ybar, gamma, L=L, prec="fp32", kernel="tc", group=g, rank=r, stream=s)
        rows = slice(sol.row0, sol.row0 + sol.rows)
        sol.set_theta(Tk[rows], Tkm1[rows], st["t_k"], st["t_kp1"])
        sol.step()
        out = dict(row0=sol.row0, T=sol.get_theta()[0], eta=sol.get_eta())
        sol.close()
        return out

    res = run_ranks(crp, world, fn)
    T = np.zeros((N, N))
    for r in res:
        T[r["row0"]:r["row0"] + r["T"].shape[0]] = r["T"]
    assert rel(T, want["Tprev"]) <= 1e-5
    assert rel(res[1]["eta"][0], want["y"]) <= 1e-5


def test_sharded_adaptive_decisions(crp):
    """Adaptive rule across ranks: the check scalars are all-reduced, so every rank takes the
    oracle's accept/reject decisions."""
    N, n, world, K = 240, 3, 2, 20
    X, ybar = crdata.random_problem(N, n, seed=9)
    gamma = 1e-3
    L = ref.lipschitz(X, gamma)
    want = oracle.papg_adaptive(X, ybar, gamma, L, K)

    def fn(r, g, s):
        sol = crp.Solver(X, ybar, gamma, L=L, prec="fp64", group=g, rank=r, stream=s, adaptive=True)
        sol.set_step_rule("adaptive", 2.0)
        trials = []
        for _ in range(K):
            sol.step()
            trials.append(sol.step_info()["trials_last"])
        out = dict(row0=sol.row0, T=sol.get_theta()[0], trials=trials)
        sol.close()
        return out

    res = run_ranks(crp, world, fn)
    for r in res:
        np.testing.assert_array_equal(r["trials"], want["trials"])
    T = np.zeros((N, N))
    for r in res:
        T[r["row0"]:r["row0"] + r["T"].shape[0]] = r["T"]
    assert rel(T, want["Tprev"]) <= 1e-11
