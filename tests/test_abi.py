"""The C-ABI boundary: libcr.so loads, exports every symbol include/cr.h declares, and its
host-only entry points behave.  No device compute is called here (CPU CI)."""
import os
import re

import numpy as np
import pytest

import crdata
import paper_1608_02227_b200 as crp
from oracle import ref

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_1608_02227_b200 import build
    build.build()
    return crp.load()


def header_functions():
    src = open(os.path.join(ROOT, "include", "cr.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cr_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_binding_exports():
    assert header_functions() == sorted(crp.EXPORTS)


def test_library_exports_every_declared_symbol(lib):
    for name in header_functions():
        assert hasattr(lib, name), name


def test_workspace_sizes_and_unsupported(lib):
    assert crp.workspace_size(50, 2, "fp64") > 2 * 64 * 256 * 8
    n4 = crp.workspace_size(16384, 40, "fp32")
    assert n4 >= 2 * 16384 * 16384 * 4
    assert crp.workspace_size(16384, 40, "fp32", rank=1, world=8) < n4 / 4
    assert crp.workspace_size(1, 2) == 0                  # N < 2
    # CR_FLAG_ADAPTIVE reserves one more Theta matrix (+ sums slot); unknown flags are rejected
    extra = crp.workspace_size(16384, 40, "fp32", flags=1) - n4
    assert 16384 * 16384 * 4 <= extra < 16384 * 16384 * 4 * 1.1
    assert crp.workspace_size(16384, 40, "fp32", flags=2) == n4          # CR_FLAG_P2P: no workspace change
    assert crp.workspace_size(16384, 40, "fp32", flags=4) == 0
    assert crp.workspace_size(100, 0) == 0                # n < 1
    assert crp.workspace_size(100, 500) == 0              # n beyond the compiled buckets
    assert crp.workspace_size(100, 4, rank=3, world=2) == 0


def test_workspace_sizes_partition(lib):
    """cr_config.nbar (Assumption 1): N % nbar == 0, nbar <= 128, shards aligned, no adaptive."""
    base = crp.workspace_size(1200, 3, "fp64")
    assert crp.workspace_size(1200, 3, "fp64", nbar=1) == base == crp.workspace_size(1200, 3, "fp64", nbar=0)
    assert crp.workspace_size(1200, 3, "fp64", nbar=12) > 0
    assert crp.workspace_size(1200, 3, "fp64", nbar=7) == 0             # N % nbar
    assert crp.workspace_size(129 * 2, 3, "fp64", nbar=129) == 0        # nbar > 128
    assert crp.workspace_size(1200, 3, "fp64", nbar=12, flags=1) == 0   # adaptive check assumes K = N
    assert crp.workspace_size(1200, 3, "fp64", nbar=12, rank=0, world=2) > 0      # S = 600
    assert crp.workspace_size(1200, 3, "fp64", nbar=24, rank=0, world=4) == 0     # S = 300
    assert crp.workspace_size(1200, 3, "fp64", nbar=-1) == 0


def test_status_strings(lib):
    assert lib.cr_status_string(0) == b"CR_OK"
    assert lib.cr_status_string(6) == b"CR_ERR_UNSUPPORTED"
    assert lib.cr_max_dim() >= 80


@pytest.mark.parametrize("N,n,seed", [(5, 1, 0), (8, 3, 1), (60, 4, 2), (700, 9, 3)])
def test_host_lanczos_matches_oracle(lib, N, n, seed):
    """libcr's structured-C^T C Lanczos (host) == the oracle's ARPACK eigsh (Eq. (lischitz))."""
    X, _ = crdata.random_problem(N, n, seed=seed)
    a = crp.lipschitz_host(X, 1e-3)
    b = ref.lipschitz(X, 1e-3)
    assert abs(a - b) <= 1e-10 * b


def test_host_lanczos_lemma4(lib):
    """Lemma 4: sigma_max(A1)^2 = 2N when X = 0."""
    for N in (3, 17, 64):
        assert abs(crp.lipschitz_host(np.zeros((N, 2)), 1.0) - 2 * N) < 1e-9 * N


def test_init_rejects_bad_arguments_without_device(lib):
    import ctypes as C
    h = C.c_void_p()
    X = np.zeros((4, 2))
    y = np.zeros(4)
    cfg = crp.binding.CrConfig(N=4, n=2, X=X.ctypes.data, ybar=y.ctypes.data, gamma=-1.0, L=0.0, prec=0,
                               kernel=0, rank=0, world=1, device=0, workspace=None, workspace_bytes=0)
    assert lib.cr_init(C.byref(cfg), C.byref(h)) == 1      # gamma <= 0
    cfg.gamma = 2.0
    assert lib.cr_init(C.byref(cfg), C.byref(h)) == 1      # gamma > 1 with L computed
    cfg.gamma, cfg.world = 1e-3, 2
    assert lib.cr_init(C.byref(cfg), C.byref(h)) == 1      # world > 1 without an NCCL id
    assert not h.value
