"""Ring-protocol stress of the tcgen05 pass (DESIGN.md §6 "ring invariants").

The pass's arithmetic does not depend on how deep its shared-memory rings are or on whether GEMM1
(S' = Xi' X_J^T, which needs only X_J and Xi') waits for the tile's Theta: every configuration must
produce Theta^K bit for bit equal to the default one, and with CR_TC_CHECK=1 the kernel tags every
slot / buffer with the tile it holds and records any consumer that finds another tile after its
barrier wait (cr_tc_check_word must stay 0).  Each configuration runs in its own process under a
timeout, so a fault or a deadlock fails one case instead of the session."""
import json
import os
import subprocess
import sys

import pytest

import crdata
from oracle import ref

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
SHAPES = [(4000, 20), (8192, 40), (4096, 80)]      # (n = 80: GEMM1 in kind::f16)
RINGS = [(2, 2, 2), (3, 2, 2), (3, 3, 3), (4, 2, 2), (5, 3, 2), (6, 2, 2), (3, 1, 1), (4, 1, 2)]


def run_case(N, n, L, env):
    e = dict(os.environ, CR_TC_CHECK="1", **env)
    r = subprocess.run([sys.executable, os.path.join(HERE, "mp", "tc_ring_case.py"), str(N), str(n), "24", repr(L)],
                       capture_output=True, text=True, timeout=180, env=e)
    assert r.returncode == 0, (env, r.stdout[-2000:], r.stderr[-2000:])
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.fixture(scope="module")
def baselines():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1608_02227_b200 import build
    build.build()
    out = {}
    for N, n in SHAPES:
        X, _ = crdata.random_problem(N, n, seed=N + n, fp32=True)
        L = ref.lipschitz(X, 1e-3)
        out[(N, n)] = (L, run_case(N, n, L, {}))
    return out


@pytest.mark.parametrize("runahead", [0, 1])
@pytest.mark.parametrize("rings", RINGS)
@pytest.mark.parametrize("shape", SHAPES)
def test_ring_depths_and_gemm1_runahead(baselines, shape, rings, runahead):
    L, base = baselines[shape]
    assert base["check"] == 0 and base["kernel"] == "tc"
    S, S1, S2 = rings
    got = run_case(*shape, L, {"CR_TC_STAGES": str(S), "CR_TC_G1STAGES": str(S1), "CR_TC_G2STAGES": str(S2),
                               "CR_TC_G1_RUNAHEAD": str(runahead)})
    assert got["check"] == 0, hex(got["check"])
    assert got["sha"] == base["sha"]
