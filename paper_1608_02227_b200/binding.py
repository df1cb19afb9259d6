"""Thin ctypes binding of libcr (include/cr.h).  Argument marshalling only.

Every step of the hot path runs in libcr's CUDA kernels; PyTorch supplies device memory
(the workspace tensor), the stream, and the process group that broadcasts the NCCL id.
There is no CPU fallback: if libcr.so is missing or no CUDA device is present, the
constructor raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcr.so")

CR_OK, CR_ERR_INVALID_ARG, CR_ERR_CUDA, CR_ERR_NCCL, CR_ERR_OOM, CR_ERR_STATE, CR_ERR_UNSUPPORTED = range(7)
PREC = {"fp32": 0, "fp64": 1}
KERNEL = {"auto": 0, "simt": 1, "tc": 2}
KERNEL_NAME = {v: k for k, v in KERNEL.items()}
STEP_RULE = {"constant": 0, "adaptive": 1, "backtrack": 2}
CR_FLAG_ADAPTIVE = 1
CR_FLAG_P2P = 2

# Symbols include/cr.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "cr_workspace_size", "cr_max_dim", "cr_nccl_get_unique_id", "cr_init", "cr_set_theta", "cr_get_theta",
    "cr_get_theta_rows", "cr_get_sums", "cr_dual_step", "cr_solve", "cr_primal", "cr_get_eta", "cr_lipschitz",
    "cr_lipschitz_host", "cr_launch_count", "cr_set_pass_timing", "cr_pass_timing", "cr_active_kernel",
    "cr_last_error", "cr_status_string", "cr_destroy", "cr_set_step_rule", "cr_step_info", "cr_set_gamma",
    "cr_continuation", "cr_local_group_create", "cr_local_group_destroy", "cr_predict", "cr_workspace_size_ex",
    "cr_partition_info", "cr_selftest_p2p", "cr_selftest_p2p_allgather", "cr_shard_rows",
    "cr_tc_check_word",
)


class CrConfig(C.Structure):
    _fields_ = [("N", C.c_int64), ("n", C.c_int32), ("X", C.c_void_p), ("ybar", C.c_void_p),
                ("gamma", C.c_double), ("L", C.c_double), ("prec", C.c_int), ("kernel", C.c_int),
                ("rank", C.c_int32), ("world", C.c_int32), ("nccl_unique_id", C.c_void_p),
                ("device", C.c_int32), ("stream", C.c_void_p), ("workspace", C.c_void_p),
                ("workspace_bytes", C.c_size_t), ("flags", C.c_int32), ("local_group", C.c_void_p),
                ("nbar", C.c_int64)]


class CrStepStats(C.Structure):
    _fields_ = [("k", C.c_int64), ("t_k", C.c_double), ("g", C.c_double), ("r_gamma", C.c_double),
                ("gap", C.c_double), ("max_violation", C.c_double), ("infeas_norm", C.c_double),
                ("nonfinite", C.c_int32)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class CrStop(C.Structure):
    _fields_ = [("report_every", C.c_int32), ("infeas_tol", C.c_double), ("gap_tol", C.c_double)]


class CrReport(C.Structure):
    _fields_ = [("iters", C.c_int64), ("converged", C.c_int32), ("last", CrStepStats)]


class CrCont(C.Structure):
    _fields_ = [("eps0", C.c_double), ("beta", C.c_double), ("kappa_gamma", C.c_double), ("stages", C.c_int32),
                ("iters", C.c_void_p), ("iters_per_stage", C.c_int64), ("stop", C.c_void_p)]


class CrContReport(C.Structure):
    _fields_ = [("stages_run", C.c_int32), ("iters_total", C.c_int64), ("gamma_last", C.c_double),
                ("L_last", C.c_double), ("last", CrStepStats)]


class CrPartitionStats(C.Structure):
    _fields_ = [("nbar", C.c_int64), ("blocks", C.c_int64), ("ipm_iters_max", C.c_int32),
                ("polish_rounds_max", C.c_int32), ("multiplier_iters_max", C.c_int32), ("failed_blocks", C.c_int64),
                ("unpolished_blocks", C.c_int64), ("warm_blocks", C.c_int64), ("factorizations", C.c_int64),
                ("solves", C.c_int64), ("products", C.c_int64), ("timed_ms", C.c_double), ("timed_launches", C.c_int64)]


class CrError(RuntimeError):
    pass


_lib = None


def load(path: str = LIB_PATH):
    """Load libcr.so (built by ``python -m paper_1608_02227_b200.build``); raise if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise CrError(f"libcr.so not found at {path}; build it with `python -m paper_1608_02227_b200.build` "
                      "(there is no CPU fallback)")
    L = C.CDLL(path)
    vp, i64, i32, d = C.c_void_p, C.c_int64, C.c_int32, C.c_double
    sig = {
        "cr_workspace_size": (C.c_size_t, [i64, i32, C.c_int, C.c_int, i32, i32, i32]),
        "cr_workspace_size_ex": (C.c_size_t, [i64, i32, C.c_int, C.c_int, i32, i32, i32, i64]),
        "cr_partition_info": (C.c_int, [vp, C.POINTER(CrPartitionStats)]),
        "cr_selftest_p2p": (C.c_int, [i32, i64, i32, vp, vp]),
        "cr_selftest_p2p_allgather": (C.c_int, [i32, i64, vp, vp]),
        "cr_max_dim": (i32, []),
        "cr_shard_rows": (i64, [i64, i32, i64]),
        "cr_tc_check_word": (C.c_uint64, [vp]),
        "cr_nccl_get_unique_id": (C.c_int, [vp]),
        "cr_init": (C.c_int, [C.POINTER(CrConfig), C.POINTER(vp)]),
        "cr_set_theta": (C.c_int, [vp, vp, vp, d, d]),
        "cr_get_theta": (C.c_int, [vp, vp, vp, C.POINTER(d), C.POINTER(d)]),
        "cr_get_theta_rows": (C.c_int, [vp, i32, i64, i64, vp]),
        "cr_get_sums": (C.c_int, [vp, i32, vp, vp, vp]),
        "cr_dual_step": (C.c_int, [vp, C.POINTER(CrStepStats)]),
        "cr_solve": (C.c_int, [vp, i64, C.POINTER(CrStop), C.POINTER(CrReport)]),
        "cr_primal": (C.c_int, [vp, vp, vp, C.POINTER(CrStepStats)]),
        "cr_get_eta": (C.c_int, [vp, vp, vp]),
        "cr_lipschitz": (d, [vp]),
        "cr_lipschitz_host": (C.c_int, [i64, i32, vp, d, C.POINTER(d)]),
        "cr_launch_count": (i64, [vp]),
        "cr_set_pass_timing": (C.c_int, [vp, i32]),
        "cr_pass_timing": (C.c_int, [vp, C.POINTER(d), C.POINTER(i64)]),
        "cr_active_kernel": (C.c_int, [vp]),
        "cr_last_error": (C.c_char_p, [vp]),
        "cr_status_string": (C.c_char_p, [C.c_int]),
        "cr_destroy": (None, [vp]),
        "cr_set_step_rule": (C.c_int, [vp, C.c_int, d, d]),
        "cr_step_info": (C.c_int, [vp, C.POINTER(d), C.POINTER(i64), C.POINTER(i64)]),
        "cr_set_gamma": (C.c_int, [vp, d, d]),
        "cr_predict": (C.c_int, [vp, vp, i64, vp]),
        "cr_local_group_create": (C.c_int, [i32, C.POINTER(vp)]),
        "cr_local_group_destroy": (None, [vp]),
        "cr_continuation": (C.c_int, [vp, C.POINTER(CrCont), C.POINTER(CrContReport)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None and a.shape != shape:
        raise ValueError(f"expected shape {shape}, got {a.shape}")
    return a


def workspace_size(N, n, prec="fp32", kernel="auto", rank=0, world=1, flags=0, nbar=1) -> int:
    return int(load().cr_workspace_size_ex(int(N), int(n), PREC[prec], KERNEL[kernel], int(rank), int(world),
                                           int(flags), int(nbar)))


def selftest_p2p(colpart) -> np.ndarray:
    """cr_selftest_p2p: colpart [world][nrb][N] fp32 -> the column sums over all ranks and rows,
    computed by the CR_FLAG_P2P push / gather kernels for `world` virtual ranks on this GPU."""
    cp = np.ascontiguousarray(colpart, dtype=np.float32)
    W, nrb, N = cp.shape
    out = np.empty(N)
    st = load().cr_selftest_p2p(int(W), int(N), int(nrb), cp.ctypes.data, out.ctypes.data)
    if st != 0:
        raise CrError(f"cr_selftest_p2p: {load().cr_status_string(st).decode()}")
    return out


def selftest_p2p_allgather(y, world) -> np.ndarray:
    """cr_selftest_p2p_allgather: y [N] fp32 -> [world][N], every virtual rank's gathered copy."""
    yy = np.ascontiguousarray(y, dtype=np.float32)
    out = np.empty((int(world), yy.shape[0]), dtype=np.float32)
    st = load().cr_selftest_p2p_allgather(int(world), int(yy.shape[0]), yy.ctypes.data, out.ctypes.data)
    if st != 0:
        raise CrError(f"cr_selftest_p2p_allgather: {load().cr_status_string(st).decode()}")
    return out


def lipschitz_host(X, gamma) -> float:
    """L = sigma_max(C)^2 / gamma by libcr's host Lanczos (Eq. (lischitz))."""
    X = _f64(X)
    out = C.c_double()
    st = load().cr_lipschitz_host(X.shape[0], X.shape[1], X.ctypes.data, float(gamma), C.byref(out))
    if st != CR_OK:
        raise CrError(f"cr_lipschitz_host: status {st}")
    return out.value


def nccl_unique_id() -> bytes:
    buf = (C.c_char * 128)()
    st = load().cr_nccl_get_unique_id(buf)
    if st != CR_OK:
        raise CrError(f"cr_nccl_get_unique_id: status {st}")
    return bytes(buf)


def shard_rows(N: int, world: int, nbar: int = 1) -> int:
    """Rows per shard, S = cr_shard_rows(N, world, nbar) (include/cr.h)."""
    return int(load().cr_shard_rows(int(N), int(world), int(nbar)))


def shard_range(N: int, rank: int, world: int, nbar: int = 1):
    """Rows [row0, row0 + rows) of Theta owned by `rank` (include/cr.h: S = cr_shard_rows)."""
    S = shard_rows(N, world, nbar)
    row0 = min(int(N), int(rank) * S)
    return row0, min(int(N), row0 + S) - row0


def broadcast_unique_id(group, device=None) -> bytes:
    """Rank 0 of `group` draws a 128-byte ncclUniqueId (cr_nccl_get_unique_id) and broadcasts it
    over torch.distributed (CPU tensor for gloo, `device` tensor for nccl)."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank(group)
    raw = nccl_unique_id() if rank == 0 else bytes(128)
    bdev = device if (device is not None and dist.get_backend(group) == "nccl") else torch.device("cpu")
    t = torch.tensor(list(raw), dtype=torch.uint8, device=bdev)
    dist.broadcast(t, src=dist.get_global_rank(group, 0), group=group)
    return bytes(t.cpu().tolist())


class LocalGroup:
    """In-process group of `world` ranks (cr_local_group_create): every rank is a Solver of this
    process, driven by its own host thread, all on one GPU (or several).  Used to run the
    row-sharded path -- all-gather of y, reduce-scatter of the column sums, scalar
    all-reduces -- end to end on a single B200.  Destroy (close) after the member Solvers."""

    def __init__(self, world: int):
        self.lib = load()
        self.world = int(world)
        h = C.c_void_p()
        st = self.lib.cr_local_group_create(self.world, C.byref(h))
        if st != CR_OK:
            raise CrError(f"cr_local_group_create({world}): status {st}")
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.lib.cr_local_group_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Solver:
    """One rank's share of the smoothed-dual P-APG solve (Fig. 2).

    X [N, n], ybar [N] are host arrays (copied).  With ``group`` (a torch.distributed
    process group of world > 1) rank r owns rows [r*S, min(N, (r+1)*S)), S = shard_rows(N, world),
    and NCCL is bootstrapped by broadcasting the unique id over ``group``.
    """

    def __init__(self, X, ybar, gamma, L=0.0, prec="fp32", kernel="auto", device=None, stream=None,
                 group=None, adaptive=False, rank=None, nbar=1, p2p=False):
        import torch
        if not torch.cuda.is_available():
            raise CrError("libcr needs a CUDA device (no CPU fallback)")
        self.lib = load()
        self.X = _f64(X)
        self.N, self.n = self.X.shape
        self.ybar = _f64(ybar, (self.N,))
        self.gamma = float(gamma)
        self.prec = prec
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else int(device))
        self.device = dev
        self.rank, self.world = 0, 1
        uid = None
        local = None
        if isinstance(group, LocalGroup):
            local = group
            self.world, self.rank = group.world, int(rank)
        elif group is not None:
            import torch.distributed as dist
            self.world = dist.get_world_size(group)
            self.rank = dist.get_rank(group)
            if self.world > 1:
                uid = (C.c_char * 128).from_buffer_copy(broadcast_unique_id(group, dev))
        self._uid = uid
        self.row0, self.rows = shard_range(self.N, self.rank, self.world, max(int(nbar), 1))
        flags = (CR_FLAG_ADAPTIVE if adaptive else 0) | (CR_FLAG_P2P if p2p else 0)
        self.nbar = int(nbar)
        nbytes = workspace_size(self.N, self.n, prec, kernel, self.rank, self.world, flags, self.nbar)
        if nbytes == 0:
            raise CrError(f"unsupported shape/precision: N={self.N} n={self.n} prec={prec} kernel={kernel} "
                          f"nbar={self.nbar}")
        import time as _time
        _t0 = _time.perf_counter()
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        self.init_ms = {"workspace_alloc": 1e3 * (_time.perf_counter() - _t0)}
        self.stream = torch.cuda.current_stream(dev) if stream is None else stream
        cfg = CrConfig(N=self.N, n=self.n, X=self.X.ctypes.data, ybar=self.ybar.ctypes.data, gamma=self.gamma,
                       L=float(L), prec=PREC[prec], kernel=KERNEL[kernel], rank=self.rank, world=self.world,
                       nccl_unique_id=C.cast(uid, C.c_void_p) if uid is not None else None,
                       device=dev.index, stream=self.stream.cuda_stream,
                       workspace=self.workspace.data_ptr(), workspace_bytes=nbytes, flags=flags,
                       local_group=local.h if local is not None else None, nbar=self.nbar)
        h = C.c_void_p()
        _t1 = _time.perf_counter()
        st = self.lib.cr_init(C.byref(cfg), C.byref(h))
        self.init_ms["cr_init"] = 1e3 * (_time.perf_counter() - _t1)     # (host-synchronous: includes L)
        if st != CR_OK:
            raise CrError(f"cr_init failed: {self.lib.cr_status_string(st).decode()}")
        self.h = h

    # ------------------------------------------------------------------ helpers
    def _check(self, st, what):
        if st != CR_OK:
            msg = self.lib.cr_last_error(self.h).decode() if self.h else ""
            raise CrError(f"{what}: {self.lib.cr_status_string(st).decode()} {msg}")

    @property
    def L(self) -> float:
        return float(self.lib.cr_lipschitz(self.h))

    @property
    def kernel(self) -> str:
        return KERNEL_NAME[int(self.lib.cr_active_kernel(self.h))]

    @property
    def launch_count(self) -> int:
        return int(self.lib.cr_launch_count(self.h))

    # ------------------------------------------------------------------ API
    def step(self, stats: bool = False):
        s = CrStepStats()
        self._check(self.lib.cr_dual_step(self.h, C.byref(s) if stats else None), "cr_dual_step")
        return s.as_dict() if stats else None

    def solve(self, iters: int, report_every: int = 0, infeas_tol: float = 1e-1, gap_tol: float = 5e-7):
        rep = CrReport()
        stop = CrStop(report_every, infeas_tol, gap_tol) if report_every > 0 else None
        self._check(self.lib.cr_solve(self.h, int(iters), C.byref(stop) if stop else None, C.byref(rep)),
                    "cr_solve")
        return dict(iters=rep.iters, converged=bool(rep.converged), last=rep.last.as_dict() if stop else None)

    def primal(self, out=None):
        """eta(Theta^k) (Theorem 1) and its diagnostics (cr_primal).  out = (y, xi): caller
        buffers (float64 C-contiguous, N and rows x n; e.g. pinned host memory) to fill instead
        of fresh arrays."""
        if out is None:
            y = np.empty(self.N)
            xi = np.empty((self.rows, self.n))
        else:
            y, xi = out
            if not (y.dtype == np.float64 and xi.dtype == np.float64 and y.flags.c_contiguous
                    and xi.flags.c_contiguous and y.shape == (self.N,) and xi.shape == (self.rows, self.n)):
                raise ValueError("primal(out=(y, xi)): float64 C-contiguous arrays of shape (N,), (rows, n)")
        s = CrStepStats()
        self._check(self.lib.cr_primal(self.h, y.ctypes.data, xi.ctypes.data, C.byref(s)), "cr_primal")
        return y, xi, s.as_dict()

    def get_eta(self):
        y = np.empty(self.N)
        xi = np.empty((self.rows, self.n))
        self._check(self.lib.cr_get_eta(self.h, y.ctypes.data, xi.ctypes.data), "cr_get_eta")
        return y, xi

    def set_theta(self, theta_km1=None, theta_km2=None, t_km1=1.0, t_k=1.0):
        shp = (self.rows, self.N)
        a = None if theta_km1 is None else _f64(theta_km1, shp)
        b = None if theta_km2 is None else _f64(theta_km2, shp)
        self._check(self.lib.cr_set_theta(self.h, None if a is None else a.ctypes.data,
                                          None if b is None else b.ctypes.data, float(t_km1), float(t_k)),
                    "cr_set_theta")

    def get_theta(self):
        a = np.empty((self.rows, self.N))
        b = np.empty((self.rows, self.N))
        tk, tk1 = C.c_double(), C.c_double()
        self._check(self.lib.cr_get_theta(self.h, a.ctypes.data, b.ctypes.data, C.byref(tk), C.byref(tk1)),
                    "cr_get_theta")
        return a, b, tk.value, tk1.value

    def get_theta_rows(self, which: int, row0: int, nrows: int):
        out = np.empty((nrows, self.N))
        self._check(self.lib.cr_get_theta_rows(self.h, int(which), int(row0), int(nrows), out.ctypes.data),
                    "cr_get_theta_rows")
        return out

    def get_sums(self, which: int = 0):
        """(r, c, Theta X) of Theta^k (which=0) or Theta^{k-1} (which=1), this rank's rows."""
        r = np.empty(self.rows)
        c = np.empty(self.rows)
        P = np.empty((self.rows, self.n))
        self._check(self.lib.cr_get_sums(self.h, int(which), r.ctypes.data, c.ctypes.data, P.ctypes.data),
                    "cr_get_sums")
        return r, c, P

    def set_step_rule(self, rule: str = "constant", upsilon: float = 2.0, s_prev: float = 0.0):
        """Step rule of Step 2: "constant" (1/L) or "adaptive" (needs adaptive=True)."""
        self._check(self.lib.cr_set_step_rule(self.h, STEP_RULE[rule], float(upsilon), float(s_prev)),
                    "cr_set_step_rule")

    def partition_info(self, check: bool = True):
        """The block projections of the last Step 1 (partition K < N): nbar, blocks, ipm_iters_max,
        polish_rounds_max, multiplier_iters_max, failed_blocks.  check: raise if any block failed."""
        ps = CrPartitionStats()
        st = self.lib.cr_partition_info(self.h, C.byref(ps))
        if check:
            self._check(st, "cr_partition_info")
        return {f: getattr(ps, f) for f, _ in ps._fields_}

    def step_info(self):
        """dict(s = s_k of the last accepted step, trials_last = l_k + 1, trials_total)."""
        sk, tl, tt = C.c_double(), C.c_int64(), C.c_int64()
        self._check(self.lib.cr_step_info(self.h, C.byref(sk), C.byref(tl), C.byref(tt)), "cr_step_info")
        return dict(s=sk.value, trials_last=tl.value, trials_total=tt.value)

    def set_gamma(self, gamma: float, L: float = 0.0):
        """New Tikhonov weight; restarts Fig. 2 at the current iterate (cr_set_gamma)."""
        self._check(self.lib.cr_set_gamma(self.h, float(gamma), float(L)), "cr_set_gamma")
        self.gamma = float(gamma)

    def continuation(self, eps0: float, beta: float, kappa_gamma: float, iters, report_every: int = 0,
                     infeas_tol: float = 1e-1, gap_tol: float = 5e-7):
        """Continuation over gamma_t = kappa_gamma eps0 / beta^t (Section 2.4.1); ``iters`` is a list of
        per-stage budgets (one stage each)."""
        its = np.ascontiguousarray(iters, dtype=np.int64)
        stop = CrStop(report_every, infeas_tol, gap_tol) if report_every > 0 else None
        p = CrCont(eps0=float(eps0), beta=float(beta), kappa_gamma=float(kappa_gamma), stages=len(its),
                   iters=its.ctypes.data, iters_per_stage=0,
                   stop=C.cast(C.pointer(stop), C.c_void_p) if stop is not None else None)
        rep = CrContReport()
        self._check(self.lib.cr_continuation(self.h, C.byref(p), C.byref(rep)), "cr_continuation")
        self.gamma = rep.gamma_last
        return dict(stages_run=rep.stages_run, iters_total=rep.iters_total, gamma_last=rep.gamma_last,
                    L_last=rep.L_last, last=rep.last.as_dict())

    def predict(self, Z):
        """f_hat(z) = max_i y_i + xi_i^T (z - x_i) at eta(Theta^k), for the rows of Z (M x n)."""
        Z = _f64(Z)
        if Z.ndim != 2 or Z.shape[1] != self.n:
            raise ValueError(f"Z must be M x {self.n}")
        out = np.empty(Z.shape[0])
        self._check(self.lib.cr_predict(self.h, Z.ctypes.data, Z.shape[0], out.ctypes.data), "cr_predict")
        return out

    @property
    def tc_check_word(self) -> int:
        """First ring-protocol violation of the tensor-core pass (CR_TC_CHECK=1 at construction)."""
        return int(self.lib.cr_tc_check_word(self.h))

    def set_pass_timing(self, on: bool):
        self._check(self.lib.cr_set_pass_timing(self.h, 1 if on else 0), "cr_set_pass_timing")

    def pass_timing(self):
        ms, n = C.c_double(), C.c_int64()
        self._check(self.lib.cr_pass_timing(self.h, C.byref(ms), C.byref(n)), "cr_pass_timing")
        return ms.value, n.value

    def close(self):
        if getattr(self, "h", None):
            self.lib.cr_destroy(self.h)
            self.h = None
        self.workspace = None          # back to torch's caching allocator

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
