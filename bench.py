#!/usr/bin/env python
"""Benchmark of the fused P-APG dual step (Fig. 2) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl ours|reference]

A step is one P-APG iteration over the whole N x N multiplier matrix of the config.
``value`` = pair-constraint updates per second for the whole job, N^2 * K / t, with t the
device time (CUDA events on the library's stream, max over ranks) of K iterations whose
inputs are already resident in HBM.  ``e2e`` is the same metric through the public API
with host buffers: Solver construction (H2D of X, ybar; Lanczos L), K iterations and the
D2H read of the estimator (y, xi) inside the timed region.  Multi-GPU: launched by
torch.distributed.run, one rank per GPU, rows of Theta sharded, NCCL all-gather of y and
reduce-scatter of column sums per iteration (fixed N: strong scaling).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DEFAULT_CONFIG = "C5"   # the largest BASELINE.json config that fits one B200 (north star N >= 16384)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None, help="timed iterations (default: the config's)")
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--kernel", default="auto", choices=["auto", "simt", "tc"])
    ap.add_argument("--step", default="constant", choices=["constant", "adaptive"],
                    help="step rule of Step 2: constant 1/L (Fig. 2, the headline) or adaptive (P:400-407)")
    ap.add_argument("--nbar", type=int, default=1,
                    help="partition block size (K = N / nbar < N, per-block projections in Step 1); 1 = all pairs")
    ap.add_argument("--p2p", action="store_true",
                    help="N > 1: reduce-scatter the column sums over NVLink peer memory (CR_FLAG_P2P)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget-s", type=float, default=20.0)
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled DURING the timed region: an NVML thread
    polling every ~2 ms (a 12 ms C4 window still gets several samples); nvidia-smi -lms 50 as
    the fallback when NVML is unavailable."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, device_index):
        self.dev = device_index
        self.proc = None
        self.nvml = None
        self.rows = []            # (sm_mhz, max_mhz, {reason names})
        self.lines = []
        self.active = False
        self.stop_ev = threading.Event()

    def start(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            uuid = None
            try:
                import torch
                uuid = str(torch.cuda.get_device_properties(self.dev).uuid)
            except Exception:
                pass
            h = None
            if uuid:
                try:
                    h = nv.nvmlDeviceGetHandleByUUID(("GPU-" + uuid) if not uuid.startswith("GPU-") else uuid)
                except Exception:
                    h = None
            if h is None:
                h = nv.nvmlDeviceGetHandleByIndex(self.dev)
            self.nvml = (nv, h)
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            bits = (nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                    nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap)
            self.bits = bits
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "50",
                 "-i", str(self.dev)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.3)
        except Exception:
            self.proc = None

    def _poll(self):
        nv, h = self.nvml
        while not self.stop_ev.is_set():
            try:
                if self.active:
                    mhz = float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.rows.append((mhz, self.max_mhz, {n for n, b in zip(self.NAMES, self.bits) if r & b}))
            except Exception:
                pass
            time.sleep(0.002)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def mark(self):
        self.active = True
        return len(self.lines)

    def stop(self, since=0):
        self.active = False
        if self.nvml is not None:
            self.stop_ev.set()
            self.t.join(timeout=2)
            rows = self.rows
            src = "nvml (2 ms polling)"
        elif self.proc is not None:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
            self.t.join(timeout=2)
            time.sleep(0.5)      # let nvidia-smi's NVML session close before anything else is timed
            raw = [l.split(", ") for l in self.lines[since:] if l.count(",") >= 7] or \
                  [l.split(", ") for l in self.lines if l.count(",") >= 7]
            rows = [(float(r[0]), float(r[1]), {self.NAMES[i] for i in range(4) if r[4 + i].strip() == "Active"})
                    for r in raw if r[0].replace(".", "").isdigit() and r[1].replace(".", "").isdigit()]
            src = "nvidia-smi -lms 50"
        else:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
        sm = sorted(r[0] for r in rows)
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": max((r[1] for r in rows), default=None),
                "reasons": sorted(set().union(*[r[2] for r in rows])) if rows else [], "samples": len(rows),
                "sm_mhz_min": sm[0] if sm else None, "source": src}


def _mem_available_gib():
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable"):
                return int(line.split()[1]) / 2**20
    except OSError:
        pass
    return 0.0


def cpu_baseline(cfg, budget_s):
    """The fp64 oracle as it stands, on this host's cores, on a bounded sample of the workload:
    full P-APG iterations of the FULL problem when its two N x N fp64 states fit in half the
    available host memory (iterations in place until ~budget_s), else of the first N'
    observations.  C1-C3 also get a 1-thread run."""
    import numpy as np
    import crdata
    import oracle
    from oracle import ref
    X, ybar = crdata.make_problem(cfg)
    full = 2 * cfg.N * cfg.N * 8 / 2**30 <= 0.5 * _mem_available_gib()
    if full:
        Np = cfg.N
    else:
        # N' so that one oracle iteration is ~budget/6 s (probe on a small prefix)
        Np = min(cfg.N, 1024)
        t0 = time.perf_counter()
        oracle.papg(X[:Np], ybar[:Np], cfg.gamma, 1e6, 1)
        dt = max(time.perf_counter() - t0, 1e-4)
        Np = int(min(cfg.N, Np * max(1.0, (budget_s / 6 / dt)) ** 0.5))
    Xs, ys = np.ascontiguousarray(X[:Np]), np.ascontiguousarray(ybar[:Np])
    L = ref.lipschitz(Xs, cfg.gamma, form="structured")
    P, Q = np.zeros((Np, Np)), np.zeros((Np, Np))
    P[0, 0] = Q[0, 0] = 0.0                           # touch: page-faulting is not oracle time
    P.fill(0.0)
    Q.fill(0.0)
    t, iters, t_used = 1.0, 0, 0.0
    while True:                                       # whole iterations, in place, until the budget
        t0 = time.perf_counter()
        t = oracle.papg(Xs, ys, cfg.gamma, L, 1, Tprev=P, Tt=Q, t=t, inplace=True)["t"]
        t_used += time.perf_counter() - t0
        iters += 1
        if t_used + t_used / iters > budget_s or iters >= 1000:
            break
    out = {"value": Np * Np * iters / t_used, "unit": "pairs/s", "cores": oracle.max_threads(),
           "kind": "oracle", "host": host_info(),
           "sample": (f"{iters} full fp64 P-APG iteration(s) of the full {cfg.name} problem (N={Np}, n={cfg.n}) "
                      if full else
                      f"{iters} full fp64 P-APG iterations on the first N'={Np} of {cfg.N} observations of "
                      f"{cfg.name} (n={cfg.n}), ") + f"from Theta^0 = 0, {t_used:.1f} s"}
    del P, Q
    if cfg.name in ("C1", "C2", "C3"):
        P1, Q1 = np.zeros((Np, Np)), np.zeros((Np, Np))
        t, it1, t1 = 1.0, 0, 0.0
        while True:
            t0 = time.perf_counter()
            t = oracle.papg(Xs, ys, cfg.gamma, L, 1, Tprev=P1, Tt=Q1, t=t, inplace=True, nthreads=1)["t"]
            t1 += time.perf_counter() - t0
            it1 += 1
            if t1 + t1 / it1 > budget_s / 2 or it1 >= 1000:
                break
        oracle.papg(Xs[:2], ys[:2], cfg.gamma, L, 1, nthreads=oracle.max_threads())   # restore the pool
        out["one_thread"] = {"value": Np * Np * it1 / t1, "unit": "pairs/s", "cores": 1,
                             "sample": f"{it1} iterations, {t1:.1f} s"}
    return out


def host_info():
    """CPU model and RAM of the host the oracle ran on (SURVEY.md §8(d) oracle timing)."""
    model, ram = None, None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
        for line in open("/proc/meminfo"):
            if line.startswith("MemTotal"):
                ram = round(int(line.split()[1]) / 2**20, 1)
                break
    except OSError:
        pass
    return {"cpu": model, "ram_gib": ram, "nproc": os.cpu_count()}


def workload(cfg):
    """The config description both arms print (the driver pairs the lines by it)."""
    return (f"{cfg.name}: N={cfg.N}, n={cfg.n}, {cfg.x_law} x, f0={cfg.f0}, gamma={cfg.gamma}, Theta0=0, "
            f"step 1/L (Lanczos)")


def run_reference(args, cfg, rank, world):
    """--impl reference: the oracle timed on host cores (rank 0 only)."""
    if rank != 0:
        return
    import numpy as np
    import crdata
    import oracle
    from oracle import ref
    K, W = args.steps or 10, args.warmup
    X, ybar = crdata.make_problem(cfg)
    # each step = one full oracle iteration on a prefix N' sized so K+W steps take ~2 minutes
    Np = min(cfg.N, 1024)
    t0 = time.perf_counter()
    oracle.papg(X[:Np], ybar[:Np], cfg.gamma, 1e6, 1)
    dt = max(time.perf_counter() - t0, 1e-4)
    Np = int(min(cfg.N, Np * max(1.0, (120.0 / (K + W) / dt)) ** 0.5))
    Xs, ys = np.ascontiguousarray(X[:Np]), np.ascontiguousarray(ybar[:Np])
    L = ref.lipschitz(Xs, cfg.gamma, form="structured")
    st = oracle.papg(Xs, ys, cfg.gamma, L, W) if W > 0 else None
    t0 = time.perf_counter()
    st = oracle.papg(Xs, ys, cfg.gamma, L, K, Tprev=None if st is None else st["Tprev"],
                     Tt=None if st is None else st["Tt"], t=1.0 if st is None else st["t"])
    t = time.perf_counter() - t0
    v = Np * Np * K / t
    line = {"metric": "pair-constraint updates/s (N^2*iters/s)", "value": v, "unit": "pairs/s", "n_gpus": world,
            "steps": K, "warmup": W, "ms_per_step": 1e3 * t / K, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": workload(cfg), "N": cfg.N, "n": cfg.n, "gamma": cfg.gamma, "iters_timed": K,
                       "kernel": "oracle (fp64, CPU)", "sampled_N": Np},
            "cpu_baseline": {"value": v, "unit": "pairs/s", "cores": oracle.max_threads(), "kind": "oracle",
                             "host": host_info(),
                             "sample": f"{K} full fp64 P-APG iterations on the first N'={Np} of {cfg.N} "
                                       f"observations of {cfg.name}"},
            "e2e": {"value": v, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    import crdata
    cfg = crdata.CONFIGS[args.config]
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, cfg, rank, world)

    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_1608_02227_b200 as crp
    from paper_1608_02227_b200 import build as _b
    _b.build()

    torch.cuda.set_device(local)
    group = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        group = dist.group.WORLD
    K = args.steps if args.steps is not None else cfg.iters
    W = max(3, args.warmup)
    X, ybar = crdata.make_problem(cfg)
    prec = cfg.prec

    adaptive = args.step == "adaptive"
    p2p = args.p2p and world > 1
    s = crp.Solver(X, ybar, cfg.gamma, prec=prec, kernel=args.kernel, group=group, adaptive=adaptive, nbar=args.nbar,
                   p2p=p2p)
    if adaptive:
        s.set_step_rule("adaptive", 2.0)
    stream = s.stream
    s.solve(W)                                            # warm-up
    torch.cuda.synchronize()
    if group is not None:
        dist.barrier()
    clk = ClockSampler(torch.cuda.current_device())
    if rank == 0:
        clk.start()
    # The timed region runs the product path: cr_solve replays one CUDA graph per iteration
    # (constant rule; per accepted iteration with a device-side trial loop for the adaptive
    # rule).  Per-kernel CUDA events would turn the graphs back into eager launches (and cost
    # C3 16% of its step), so the fused pass's launch duration for the roofline is measured with
    # events on the launching stream in a window of the same solver right after the timed region
    # (same kernel, same state size, warm).
    s.set_pass_timing(False)
    l0 = s.launch_count
    tr0 = s.step_info()["trials_total"]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if group is not None:
        dist.barrier()
    mark = clk.mark()
    e0.record(stream)
    s.solve(K)
    e1.record(stream)
    torch.cuda.synchronize()
    if group is not None:
        dist.barrier()
    clocks = clk.stop(mark) if rank == 0 else None
    t_ms = e0.elapsed_time(e1)
    launches = s.launch_count - l0
    trials = s.step_info()["trials_total"] - tr0
    Kp = min(K, 20 if adaptive else 200)
    ps0 = s.partition_info(check=False) if args.nbar > 1 else None
    s.set_pass_timing(True)
    s.solve(Kp)
    pass_ms, pass_n = s.pass_timing()
    s.set_pass_timing(False)
    if group is not None:
        t = torch.tensor([t_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_ms = float(t.item())

    # what the JSON line needs from the device-timed solver; then release it (its workspace
    # returns to torch's cache, so the e2e solver below does not pay a fresh multi-GB cudaMalloc
    # whose cost depends on what the previous process left for the driver to scrub)
    s_rows, s_kernel = s.rows, s.kernel
    ps1 = s.partition_info(check=False) if args.nbar > 1 else None      # after the event window
    if not args.no_e2e:
        s.primal()        # warm-up of the primal path (one-time CUDA module loading), untimed
    s.close()
    torch.cuda.synchronize()

    # end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        Xp = torch.from_numpy(X).pin_memory().numpy()
        yp = torch.from_numpy(ybar).pin_memory().numpy()
        row0, rows = crp.binding.shard_range(cfg.N, rank, world)
        yo_pin = torch.empty(cfg.N, dtype=torch.float64).pin_memory().numpy()
        xio_pin = torch.empty((rows, cfg.n), dtype=torch.float64).pin_memory().numpy()
        torch.cuda.synchronize()
        if group is not None:
            dist.barrier()
        t0 = time.perf_counter()
        s2 = crp.Solver(Xp, yp, cfg.gamma, prec=prec, kernel=args.kernel, group=group, adaptive=adaptive,
                        nbar=args.nbar, p2p=p2p)
        if adaptive:
            s2.set_step_rule("adaptive", 2.0)
        torch.cuda.synchronize()
        t_init = time.perf_counter() - t0
        init_detail = getattr(s2, "init_ms", None)
        s2.solve(K)
        torch.cuda.synchronize()
        t_solve = time.perf_counter() - t0 - t_init
        y, xi, _ = s2.primal(out=(yo_pin, xio_pin))
        torch.cuda.synchronize()
        te = time.perf_counter() - t0
        if group is not None:
            t = torch.tensor([te], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            te = float(t.item())
        s2.close()
        e2e = {"value": cfg.N * cfg.N * K / te, "unit": "pairs/s",
               "h2d_bytes_per_step": (X.nbytes + ybar.nbytes) / K,
               "d2h_bytes_per_step": (y.nbytes + xi.nbytes + 64) / K,
               "timed": "Solver(X, ybar) [H2D from pinned host + Lanczos L + init] + solve(K) + "
                        "primal() [eta(Theta^K) + diagnostics, D2H of y, xi into pinned host buffers]; "
                        "process warmed by the device-timed solver (incl. one untimed primal)",
               "split_ms": {"init": 1e3 * t_init, "solve": 1e3 * t_solve, "primal": 1e3 * (te - t_init - t_solve),
                            "init_detail": init_detail}}

    if rank != 0:
        if group is not None:
            dist.destroy_process_group()
        return
    value = cfg.N * cfg.N * K / (t_ms / 1e3)
    bpp = 24 if prec == "fp64" else 12
    per_launch_bytes = bpp * s_rows * cfg.N
    avg_pass_s = (pass_ms / max(pass_n, 1)) / 1e3
    peak, peak_kind = peaks()
    achieved = per_launch_bytes / avg_pass_s / 1e9
    traffic = None
    tfile = os.path.join(ROOT, "profiles", f"traffic_{cfg.name}_{s_kernel}.json")
    if os.path.exists(tfile):
        try:
            traffic = json.load(open(tfile)).get("bytes_per_launch")
        except Exception:
            traffic = None
    line = {
        "metric": "pair-constraint updates/s (N^2*iters/s)",
        "value": value, "unit": "pairs/s", "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": t_ms / K, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64" if prec == "fp64" else "f32", "data": "synthetic",
        "config": {"workload": workload(cfg),
                   "N": cfg.N, "n": cfg.n, "gamma": cfg.gamma, "iters_timed": K,
                   "kernel": s_kernel, "parallelism": f"rows{world}", "step_rule": args.step,
                   "column_reduce_scatter": "peer-memory (CR_FLAG_P2P)" if p2p else ("nccl" if world > 1 else "none"),
                   **({"nbar": args.nbar, "partition": f"K = N / {args.nbar} blocks; N^2 - N*nbar pairs dualized; "
                       "Step 1 = per-block fp64 projections (block_ipm, warm started)"} if args.nbar > 1 else {}),
                   "l2": f"inputs larger than L2: Theta state {2 * bpp // 3 * cfg.N * cfg.N / 2**30:.2f} GiB "
                         f"streamed per iteration vs 126 MB L2" if cfg.N >= 8192 else "L2-resident config"},
        "hbm_gbs_algorithmic": achieved,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                     "kernel": f"fused pair pass ({s_kernel})", "bytes_per_launch": per_launch_bytes,
                     "avg_launch_ms": avg_pass_s * 1e3, "pass_share_of_step": avg_pass_s * 1e3 / max(t_ms / K, 1e-9),
                     "timing": f"pass launches event-timed in a {Kp}-iteration window after the timed region "
                               f"({pass_n} launches); the timed region replays the CUDA graphs"},
        "gpu_launches": launches,
        **({"adaptive": {"trials_per_iter": trials / K, "passes_timed": pass_n,
                         "note": "value counts accepted iterations; every trial is one fused pass; the "
                                 "timed region replays one CUDA graph per iteration (WHILE node over "
                                 "trials); roofline from the 20-iteration event-timed window after it"}}
           if adaptive else {}),
        "clocks": clocks,
        "e2e": e2e,
    }
    if args.nbar > 1:
        # the dominant kernel is the per-block projection: fp64 CUDA-core arithmetic, counted
        # with the work model of DESIGN.md §9 (FMAs per factorization / solve / product)
        nb_, n_ = args.nbar, cfg.n
        f_fact = nb_ * (n_ * n_ * nb_ + n_ * nb_ + n_ ** 3 / 6) + nb_ ** 3 * n_ / 2 + nb_ ** 3 / 6 + nb_ * nb_
        f_solve = 2 * nb_ * n_ * n_ + 3 * nb_ * nb_ * n_ + nb_ * nb_
        f_prod = nb_ * nb_ * n_
        fmas = (f_fact * (ps1["factorizations"] - ps0["factorizations"]) + f_solve * (ps1["solves"] - ps0["solves"])
                + f_prod * (ps1["products"] - ps0["products"]))
        bp_s = ps1["timed_ms"] / 1e3
        tf = 2 * fmas / max(bp_s, 1e-12) / 1e12
        fp64_peak = 33.48
        line["roofline_pass"] = line["roofline"]
        line["roofline"] = {"bound": "alu", "achieved": tf, "peak": fp64_peak, "unit": "TFLOP/s", "frac": tf / fp64_peak,
                            "traffic": None, "peak_kind": "measured fp64 FFMA (tools/probe/fprate.cu, profiles/r01/fprate.txt)",
                            "kernel": "block_ipm (per-block projections)", "flops_timed": 2 * fmas,
                            "avg_launch_ms": ps1["timed_ms"] / max(ps1["timed_launches"], 1),
                            "share_of_step": (ps1["timed_ms"] / max(ps1["timed_launches"], 1)) / max(t_ms / K, 1e-9),
                            "timing": f"block_ipm launches event-timed in the {Kp}-iteration window after the "
                                      "timed region; work counted over the same window"}
        line["partition_stats"] = ps1
    if not args.no_cpu_baseline and world == 1 and args.nbar == 1:
        line["cpu_baseline"] = cpu_baseline(cfg, args.cpu_budget_s)
    print(json.dumps(line), flush=True)
    s.close()
    if group is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
