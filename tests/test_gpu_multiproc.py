"""Row-sharded path across GPUs (north star (c)): world = 2 / 4 / 8 processes,
one per GPU, NCCL (and CR_FLAG_P2P peer memory) exchanges of y' and the column sums, against the
fp64 oracle (Fig. 2).  Skipped unless the box has at least `world` GPUs -- this pool
lends one GPU per call, where tests/test_gpu_sharded_local.py (in-process ranks) and
tests/test_gpu_nccl1.py / test_gpu_p2p.py (1-rank NCCL, cooperative self-tests) cover the same
code; these run as they are on the first multi-GPU box."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import crdata
import oracle
from oracle import ref

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _gpus():
    try:
        import torch
        return torch.cuda.device_count() if torch.cuda.is_available() else 0
    except Exception:
        return 0


def _port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def run_ranks(world, cfg_name, N, K, p2p, L, tmp):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(HERE, "mp", "worker.py"), cfg_name, str(N), str(K), "1" if p2p else "0", str(tmp), repr(L)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    parts = [dict(np.load(os.path.join(tmp, f"rank{q}.npz"))) for q in range(world)]
    T = np.concatenate([p["T"] for p in parts])
    xi = np.concatenate([p["xi"] for p in parts])
    return T, parts[0]["y"], xi, parts


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("cfg_name,N", [("C3", 4000), ("C4", 4096)])
@pytest.mark.parametrize("p2p", [False, True])
def test_sharded_across_gpus_matches_oracle(tmp_path, world, cfg_name, N, p2p):
    if _gpus() < world:
        pytest.skip(f"needs {world} GPUs ({_gpus()} visible)")
    cfg = crdata.CONFIGS[cfg_name]
    X, ybar = crdata.make_problem(cfg, N=N)
    L = ref.lipschitz(X, cfg.gamma)
    K = 6
    T, y, xi, parts = run_ranks(world, cfg_name, N, K, p2p, L, tmp_path)
    o = oracle.papg(X, ybar, cfg.gamma, L, K)
    yo, xio = oracle.eta(X, ybar, cfg.gamma, o["Tprev"])
    so = oracle.stats(X, ybar, cfg.gamma, o["Tprev"], yo, xio)
    rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
    assert rel(T, o["Tprev"]) <= 1e-5
    assert rel(y, yo) <= 1e-5 and rel(xi, xio) <= 1e-5
    for p in parts:                       # every rank reports the all-reduced diagnostics
        assert abs(float(p["r_gamma"]) - so["r_gamma"]) <= 1e-5 * abs(so["r_gamma"])
        assert abs(float(p["max_violation"]) - so["max_violation"]) <= 1e-4 * abs(so["max_violation"])
