"""Multi-process (world size 2, gloo, CPU) tests of the row-sharded path's host logic.

The GPU library shards Theta by row blocks (include/cr.h: rank p owns rows [pS, min(N,(p+1)S)),
S = ceil(N/world)) and exchanges, per iteration, an all-gather of y and a reduce-scatter of
the column sums.  Here two gloo ranks run exactly that decomposition of one
P-APG iteration (Fig. 2) in fp64 numpy -- each rank computing only its own rows'
quantities and exchanging only the two length-N vectors -- and the assembled result must
equal the unsharded fp64 oracle step.  The NCCL-id bootstrap the binding uses is also
exercised over gloo.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import crdata
import oracle


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, N, n, out_dir):
    import torch
    import torch.distributed as dist
    from paper_1608_02227_b200.binding import shard_range, broadcast_unique_id
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        X, ybar = crdata.random_problem(N, n, seed=3)
        gamma, L = 1e-2, 250.0
        Tprev = crdata.random_theta(N, seed=4, scale=1e-3)       # theta^{k-1}
        Tt = crdata.random_theta(N, seed=5, scale=1e-3)          # theta~^k
        row0, rows = shard_range(N, rank, world)
        S = -(-N // world)
        mine = slice(row0, row0 + rows)
        # --- this rank's sums of theta~ over its rows (row-local) + column partials over its rows
        Tt_m = Tt[mine]
        r = Tt_m.sum(axis=1) - np.diag(Tt[mine, mine]) if rows else np.zeros(0)
        cpart = np.zeros(world * S)
        cpart[:N] = Tt_m.sum(axis=0) - np.concatenate(
            [np.zeros(row0), np.diag(Tt[mine, mine]), np.zeros(N - row0 - rows)]) if rows else 0.0
        P = Tt_m @ X
        # --- reduce-scatter of the column sums (gloo: all_reduce + own slice)
        ct = torch.from_numpy(cpart)
        dist.all_reduce(ct)
        c = ct.numpy()[row0:row0 + rows]
        # --- Step 1 on own rows: y = ybar + c - r, xi_i = (r_i x_i - (Theta X)_i)/gamma
        y_m = ybar[mine] + c - r
        xi_m = (r[:, None] * X[mine] - P) / gamma
        # --- all-gather of y
        parts = [torch.zeros(S, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(np.pad(y_m, (0, S - rows))))   # S per rank, padded
        y = torch.cat(parts).numpy()[:N]
        # --- Step 2 on own rows x all columns
        R = y[None, :] - y_m[:, None] + (xi_m * X[mine]).sum(1)[:, None] - xi_m @ X.T
        Tk = np.maximum(0.0, Tt_m - R / L)
        Tk[np.arange(rows), np.arange(row0, row0 + rows)] = 0.0
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), Tk=Tk, y=y, xi=xi_m, row0=row0)
        # --- NCCL unique id bootstrap over the process group
        uid = broadcast_unique_id(dist.group.WORLD)
        with open(os.path.join(out_dir, f"uid{rank}.bin"), "wb") as f:
            f.write(uid)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("N,n", [(37, 3), (64, 2)])
def test_row_sharded_step_equals_oracle(tmp_path, N, n):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), N, n, str(tmp_path)), nprocs=world, join=True)
    X, ybar = crdata.random_problem(N, n, seed=3)
    Tprev = crdata.random_theta(N, seed=4, scale=1e-3)
    Tt = crdata.random_theta(N, seed=5, scale=1e-3)
    want = oracle.papg(X, ybar, 1e-2, 250.0, 1, Tprev=Tprev, Tt=Tt, t=3.0)
    Tk = np.zeros((N, N))
    for rank in range(world):
        d = np.load(tmp_path / f"r{rank}.npz")
        r0 = int(d["row0"])
        Tk[r0:r0 + d["Tk"].shape[0]] = d["Tk"]
        np.testing.assert_allclose(d["y"], want["y"], rtol=0, atol=1e-12)
        np.testing.assert_allclose(d["xi"], want["xi"][r0:r0 + d["xi"].shape[0]], rtol=0, atol=1e-9)
    np.testing.assert_allclose(Tk, want["Tprev"], rtol=0, atol=1e-15)
    u0 = (tmp_path / "uid0.bin").read_bytes()
    u1 = (tmp_path / "uid1.bin").read_bytes()
    assert len(u0) == 128 and u0 == u1


def test_shard_ranges_cover_rows_once():
    from paper_1608_02227_b200.binding import shard_range
    import paper_1608_02227_b200 as crp
    crp.load()
    for N in (2, 7, 1000, 16384, 65537):
        for world in (1, 2, 3, 4, 8):
            rows = [shard_range(N, r, world) for r in range(world)]
            assert sum(k for _, k in rows) == N
            S = crp.binding.shard_rows(N, world)
            assert all(rows[r][0] == min(N, r * S) for r in range(world))
            assert all(rows[r][0] + rows[r][1] == rows[r + 1][0] for r in range(world - 1))
            # every rank gets a workspace (possibly for zero rows) and ranks never overlap
            for r in range(world):
                assert crp.workspace_size(N, 5, rank=r, world=world) > 0


def test_shard_rows_padded_to_column_blocks():
    """cr_shard_rows (include/cr.h): with world > 1 the shard is ceil(N/world) rounded up to the
    128-column block of the column-sum exchange whenever every rank keeps >= 1 row -- so the
    peer-memory path (CR_FLAG_P2P) covers C3 (N = 4000) at 2/4/8 ranks; a partition keeps
    ceil(N/world) (S % nbar == 0 is required instead); world 1 is the whole problem."""
    import paper_1608_02227_b200 as crp
    sr = crp.binding.shard_rows
    for N in (4000, 16384, 65536):
        for W in (2, 4, 8):
            S = sr(N, W)
            assert S % 128 == 0 and (W - 1) * S < N and S >= -(-N // W)
    assert sr(4000, 8) == 512 and sr(4000, 4) == 1024 and sr(4000, 2) == 2048
    assert sr(300, 4) == 75                      # padding would leave rank 3 without rows
    assert sr(1000, 1) == 1000 and sr(4000, 4, 100) == 1000
    for N in range(2, 700, 7):
        for W in (2, 3, 5, 8):
            S = sr(N, W)
            assert S >= -(-N // W) and (W - 1) * S < N or S == -(-N // W)
