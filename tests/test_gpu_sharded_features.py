"""The row-sharded path (world > 1, in-process local group on one GPU) with the
widened features: the adaptive step rule (its check sums are all-reduced across ranks), the
monotone backtracking variant and continuation over gamma -- each assembled from the ranks and
compared with the fp64 oracle like the single-rank runs (the partition K < N: see
tests/test_gpu_partition.py::test_partition_sharded_local_group)."""
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
    import torch
    g = crp.LocalGroup(world)
    out, errs = [None] * world, []

    def body(r):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                out[r] = fn(r, g, st)
            st.synchronize()
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


def assemble(res, N):
    T = np.zeros((N, N))
    for r in res:
        T[r["row0"]:r["row0"] + r["T"].shape[0]] = r["T"]
    return T


@pytest.mark.parametrize("rule,N,n,prec,kernel,world,K,tol", [
    ("adaptive", 97, 3, "fp64", "auto", 2, 25, 1e-11),
    ("adaptive", 1000, 20, "fp32", "tc", 3, 20, 2e-5),
    ("backtrack", 300, 4, "fp64", "auto", 2, 30, 1e-11),
])
def test_sharded_step_rules_match_oracle(crp, rule, N, n, prec, kernel, world, K, tol):
    X, ybar = crdata.random_problem(N, n, seed=N + 7, fp32=prec == "fp32")
    gamma = 1e-3
    L = ref.lipschitz(X, gamma)
    s0 = L if rule == "adaptive" else L / 16
    want = oracle.papg_adaptive(X, ybar, gamma, s0, K, ups=2.0, backtrack=rule == "backtrack")

    def fn(r, g, st):
        sol = crp.Solver(X, ybar, gamma, L=L, prec=prec, kernel=kernel, group=g, rank=r, stream=st, adaptive=True)
        sol.set_step_rule(rule, 2.0, s_prev=0.0 if rule == "adaptive" else s0)
        trials = []
        for _ in range(K):
            sol.step()
            trials.append(sol.step_info()["trials_last"])
        out = dict(row0=sol.row0, T=sol.get_theta()[0], trials=trials, s=sol.step_info()["s"])
        sol.close()
        return out

    res = run_ranks(crp, world, fn)
    for r in res:
        np.testing.assert_array_equal(r["trials"], want["trials"])     # every rank took the same decisions
        assert r["s"] == pytest.approx(want["s_hist"][-1], rel=1e-15)
    assert rel(assemble(res, N), want["Tprev"]) <= tol


def test_sharded_continuation_matches_oracle(crp):
    N, n, world, iters = 150, 3, 3, [20, 20, 20]
    X, ybar = crdata.random_problem(N, n, seed=12)
    gamma0 = 1e-2
    L0 = ref.lipschitz(X, gamma0)
    want = oracle.continuation(X, ybar, L0 * gamma0, eps0=1e-1, beta=4.0, kappa_gamma=0.1, iters=iters)

    def fn(r, g, st):
        sol = crp.Solver(X, ybar, gamma0, L=L0, prec="fp64", group=g, rank=r, stream=st)
        rep = sol.continuation(1e-1, 4.0, 0.1, iters)
        y, xi, stt = sol.primal()
        out = dict(row0=sol.row0, T=sol.get_theta()[0], rep=rep, y=y, stats=stt)
        sol.close()
        return out

    res = run_ranks(crp, world, fn)
    assert all(r["rep"]["stages_run"] == len(iters) for r in res)
    assert rel(assemble(res, N), want[-1]["Theta"]) <= 1e-11
    assert rel(res[0]["y"], want[-1]["y"]) <= 1e-11
    so = oracle.stats(X, ybar, want[-1]["gamma"], want[-1]["Theta"], want[-1]["y"], want[-1]["xi"])
    assert abs(res[0]["stats"]["r_gamma"] - so["r_gamma"]) <= 1e-11 * abs(so["r_gamma"])
