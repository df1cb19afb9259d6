"""CR_FLAG_P2P: the column-sum reduce-scatter over peer memory.

Across GPUs it cannot run on this pool's single GPU; what runs here is (1) the protocol itself
-- the production column-sum blocks pushing into owner slabs with system-scope releases and the
owner gathers acquiring them -- for W virtual ranks in ONE cooperative launch
(cr_selftest_p2p), checked against plain column sums; (2) the production wiring end to end on a
1-rank NCCL communicator (CR_FORCE_NCCL): reduce kernel push, gather kernel, epochs across CUDA
graph replays, bit-identical to the NCCL reduce-scatter path."""
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


@pytest.mark.parametrize("W,N,nrb", [(1, 640, 8), (2, 2048, 16), (3, 766, 5), (4, 4096, 32), (8, 8192, 4)])
def test_selftest_protocol_matches_column_sums(crp, W, N, nrb):
    rng = np.random.default_rng(W * 1000 + N)
    cp = rng.random((W, nrb, N), dtype=np.float32)
    c = crp.selftest_p2p(cp)
    want = cp.astype(np.float64).sum(axis=(0, 1))
    np.testing.assert_allclose(c, want, rtol=1e-13, atol=0)


@pytest.mark.parametrize("W,N", [(1, 300), (2, 1000), (3, 1001), (5, 4097), (8, 20000)])
def test_selftest_allgather_protocol(crp, W, N):
    y = np.random.default_rng(W + N).random(N, dtype=np.float32)
    out = crp.selftest_p2p_allgather(y, W)
    for q in range(W):
        np.testing.assert_array_equal(out[q], y)


def test_selftest_rejects_straddling_blocks(crp):
    with pytest.raises(crp.CrError):
        crp.selftest_p2p(np.zeros((4, 2, 300), dtype=np.float32))       # S = ceil(300/4) = 75: padding to
                                                                        # 128 would leave rank 3 no rows


@pytest.mark.parametrize("N,n,prec,kernel", [(1024, 20, "fp32", "tc"), (512, 5, "fp32", "simt"),
                                             (320, 3, "fp64", "auto")])
def test_p2p_one_rank_nccl_equals_nccl_reduce_scatter(crp, monkeypatch, N, n, prec, kernel):
    monkeypatch.setenv("CR_FORCE_NCCL", "1")
    X, ybar = crdata.random_problem(N, n, seed=N + n, fp32=prec == "fp32")
    gamma = 1e-3
    L = ref.lipschitz(X, gamma)
    out = []
    for p2p in (False, True):
        s = crp.Solver(X, ybar, gamma, L=L, prec=prec, kernel=kernel, p2p=p2p)
        s.solve(7)                              # graph replays: the gather's epochs advance
        s.step()                                # and an eager step
        T, T1, tk, _ = s.get_theta()
        y, xi, st = s.primal()
        out.append((T, T1, y, xi, st["r_gamma"]))
        s.close()
    for a, b in zip(out[0], out[1]):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("mode", ["adaptive", "partition"])
def test_p2p_one_rank_nccl_adaptive_and_partition(crp, monkeypatch, mode):
    """The adaptive rule's trial prologues and the partition's refreshed prologue push y' too."""
    monkeypatch.setenv("CR_FORCE_NCCL", "1")
    N, n = 256, 3
    X, ybar = crdata.random_problem(N, n, seed=3)
    gamma = 1e-2
    L = ref.lipschitz(X, gamma)
    out = []
    for p2p in (False, True):
        if mode == "adaptive":
            s = crp.Solver(X, ybar, gamma, L=L, prec="fp64", adaptive=True, p2p=p2p)
            s.set_step_rule("adaptive", 2.0)
        else:
            s = crp.Solver(X, ybar, gamma, L=L, prec="fp64", nbar=16, p2p=p2p)
        s.solve(6)
        s.step()
        out.append(s.get_theta()[0])
        s.close()
    np.testing.assert_array_equal(out[0], out[1])


def test_p2p_rejects_unaligned_shards(crp, monkeypatch):
    monkeypatch.setenv("CR_FORCE_NCCL", "1")
    X, ybar = crdata.random_problem(300, 3, seed=2, fp32=True)      # S = 300: not a multiple of 128
    with pytest.raises(crp.CrError):
        crp.Solver(X, ybar, 1e-3, L=1.0, prec="fp32", p2p=True)


def test_p2p_flag_needs_nccl(crp):
    X, ybar = crdata.random_problem(256, 3, seed=1)
    with pytest.raises(crp.CrError):
        crp.Solver(X, ybar, 1e-3, L=1.0, p2p=True)          # world 1 without CR_FORCE_NCCL
