"""Full-size K-iteration parity records: the GPU path (libcr through the C
ABI, the bench's launch configuration: cr_solve's CUDA-graph replays) against the fp64 oracle
(oracle/papg_oracle.c, Fig. 2) on the same seeded config, same L, K iterations from
Theta^0 = 0; the estimator eta(Theta^K) (Theorem 1) and its diagnostics
compared.

    python tools/full_parity.py oracle C4 1000     # oracle leg (CPU only; ~6n flops/pair/iter)
    python tools/full_parity.py gpu C4 1000        # GPU leg: reads the oracle leg's cache
    python tools/full_parity.py both C5 200        # both in one process (the GPU box's host)

The oracle leg writes gpurun_in/oracle_<cfg>_K<K>.npz (git-ignored; it travels to the GPU box
with the gpurun snapshot): L, eta(Theta^K) = (y, xi), the stats, and sampled rows of Theta^K.
Every stored value comes from oracle/ only.  The GPU leg writes profiles/r02/parity_<cfg>_K<K>.json.
"""
from __future__ import annotations

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import crdata  # noqa: E402

CACHE = os.path.join(ROOT, "gpurun_in")
OUT = os.path.join(ROOT, "profiles", "r02")


def sample_rows(N):
    """Rows compared element by element: both ends, tile boundaries, and a seeded spread."""
    rng = np.random.default_rng(2024)
    fixed = [0, 1, 127, 128, 129, N // 2 - 1, N // 2, N - 129, N - 128, N - 1]
    rows = np.unique(np.concatenate([fixed, rng.choice(N, size=min(N, 54), replace=False)]))
    return rows.astype(np.int64)


def oracle_leg(cfg, K):
    import oracle
    from oracle import ref
    X, ybar = crdata.make_problem(cfg)
    N = cfg.N
    t0 = time.perf_counter()
    L = ref.lipschitz(X, cfg.gamma)
    tL = time.perf_counter() - t0
    Tprev = np.zeros((N, N))
    Tt = np.zeros((N, N))
    t0 = time.perf_counter()
    st = oracle.papg(X, ybar, cfg.gamma, L, K, Tprev=Tprev, Tt=Tt, t=1.0, inplace=True)
    t_iter = time.perf_counter() - t0
    del Tt
    st["Tt"] = None
    y, xi = oracle.eta(X, ybar, cfg.gamma, Tprev)
    so = oracle.stats(X, ybar, cfg.gamma, Tprev, y, xi)
    rows = sample_rows(N)
    rec = dict(L=L, y=y, xi=xi, rows=rows, theta_rows=Tprev[rows].copy(), t=st["t"],
               stats=np.array([so[k] for k in ("r_gamma", "g", "gap", "max_violation", "infeas_norm")]),
               nnz=np.count_nonzero(Tprev), seconds=t_iter, lanczos_s=tL, threads=oracle.max_threads())
    os.makedirs(CACHE, exist_ok=True)
    path = os.path.join(CACHE, f"oracle_{cfg.name}_K{K}.npz")
    np.savez(path, **rec)
    print(f"oracle {cfg.name} K={K}: {t_iter:.1f} s on {oracle.max_threads()} threads; stats {so}", flush=True)
    return path


def rel(a, b):
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def gpu_leg(cfg, K):
    import torch
    import paper_1608_02227_b200 as crp
    d = np.load(os.path.join(CACHE, f"oracle_{cfg.name}_K{K}.npz"))
    X, ybar = crdata.make_problem(cfg)
    L = float(d["L"])
    s = crp.Solver(X, ybar, cfg.gamma, L=L, prec=cfg.prec)
    s.solve(K)
    torch.cuda.synchronize()
    y, xi, sg = s.primal()
    rows = d["rows"]
    Tg = np.concatenate([s.get_theta_rows(0, int(r), 1) for r in rows])
    kernel = s.kernel
    s.close()
    To = d["theta_rows"]
    names = ("r_gamma", "g", "gap", "max_violation", "infeas_norm")
    so = dict(zip(names, (float(v) for v in d["stats"])))
    err = {k: abs(sg[k] - so[k]) / max(abs(so[k]), 1e-300) for k in names}
    floor = None
    fpath = os.path.join(OUT, f"floor_{cfg.name}.jsonl")
    if os.path.exists(fpath):
        for line in open(fpath):
            r = json.loads(line)
            if r.get("K") == K:
                floor = r
    out = {
        "config": cfg.name, "N": cfg.N, "n": cfg.n, "K": K, "gamma": cfg.gamma, "L": L, "kernel": kernel,
        "prec": cfg.prec,
        "what": "K iterations from Theta^0 = 0 (cr_solve graph replays) vs the fp64 oracle (Fig. 2, P:377-397); "
                "eta(Theta^K) and its diagnostics (Theorem 1 P:241-247, P:1104-1106)",
        "objective_rel_err": err["r_gamma"], "max_violation_rel_err": err["max_violation"],
        "g_rel_err": err["g"], "gap_rel_err": err["gap"], "infeas_norm_rel_err": err["infeas_norm"],
        "gpu": {k: float(sg[k]) for k in names}, "oracle": so,
        "y_rel_err": rel(y, d["y"]), "xi_rel_err": rel(xi, d["xi"]),
        "theta_rows": {"rows": len(rows), "frobenius_rel_err": rel(Tg, To),
                       "max_abs_err_over_max_abs": float(np.abs(Tg - To).max() / max(np.abs(To).max(), 1e-300)),
                       "nnz_oracle": int(np.count_nonzero(To)), "nnz_gpu": int(np.count_nonzero(Tg))},
        "north_star_tol": 1e-4,
        "objective_within_1e-4": err["r_gamma"] <= 1e-4,
        "max_violation_within_1e-4": err["max_violation"] <= 1e-4,
        "fp32_storage_floor": floor,
        "oracle_seconds": float(d["seconds"]), "oracle_threads": int(d["threads"]),
    }
    for od in (OUT, os.path.join(ROOT, "gpurun_out")):    # (gpurun_out: merged back from a GPU box)
        os.makedirs(od, exist_ok=True)
        with open(os.path.join(od, f"parity_{cfg.name}_K{K}.json"), "w") as f:
            json.dump(out, f, indent=1)
    print(json.dumps(out), flush=True)
    return out


if __name__ == "__main__":
    leg, name = sys.argv[1], sys.argv[2]
    cfg = crdata.CONFIGS[name]
    K = int(sys.argv[3]) if len(sys.argv) > 3 else cfg.iters
    if leg in ("oracle", "both"):
        oracle_leg(cfg, K)
    if leg in ("gpu", "both"):
        gpu_leg(cfg, K)
