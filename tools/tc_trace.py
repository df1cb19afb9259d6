"""Per-tile timeline of CTA 0 of the tensor-core pass (debug; CR_TC_TRACE).

    CR_NVCC_EXTRA=-DCR_TC_TRACE_BUILD python -c "import paper_1608_02227_b200.build as b; b.build(force=True)"
    python tools/tc_trace.py C3 [steps]

The timeline events exist only in a trace build (-DCR_TC_TRACE_BUILD; production builds compile
them out -- they cost the pass several percent), so build one in a copy of the tree.

Runs `steps` eager dual steps of the config's problem (the last one's timeline is kept) and
prints, per tile u of CTA 0, the clock64 offsets (in cycles from kernel entry) of each role's
events (see TC_TRACE in kernels/pass_tc.cu):
  producer: Theta issue (P), X1 issue, X2 issue; GEMM1: start, waits passed (G1w), commit (G1c);
  GEMM2: start, waits passed, commit; storer: st_full passed (STf), slot read (STr);
  epilogue: start, Theta landed (Et), D1 ready (Ed), at_empty, compute done (Ec), barrier, end (Ee).
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    cfgname = sys.argv[1] if len(sys.argv) > 1 else "C3"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 12
    out = os.path.abspath(os.environ.get("TRACE_OUT", f"gpurun_out/trace_{cfgname}.bin"))
    os.makedirs(os.path.dirname(out), exist_ok=True)
    os.environ["CR_TC_TRACE"] = out
    import crdata
    import paper_1608_02227_b200 as crp
    cfg = crdata.CONFIGS[cfgname]
    X, ybar = crdata.make_problem(cfg)
    s = crp.Solver(X, ybar, cfg.gamma, prec="fp32")
    for _ in range(steps):
        s.step()
    s.close()
    raw = np.fromfile(out, dtype=np.uint64).astype(np.int64)
    t = raw[:5 * 256 * 8].reshape(5, 256, 8)
    cta = raw[5 * 256 * 8:].reshape(-1, 4)
    cta = cta[cta[:, 0] > 0]
    if len(cta):
        g0 = cta[:, 0].min()
        ent, pdl, ex, U = (cta[:, 0] - g0) / 1e3, (cta[:, 1] - g0) / 1e3, (cta[:, 2] - g0) / 1e3, cta[:, 3]
        dur = ex - pdl
        print(f"{cfgname}: {len(cta)} CTAs; entry spread {ent.max():.2f} us, predecessor done {pdl.min():.2f}-{pdl.max():.2f} us, "
              f"exit {ex.min():.2f}-{ex.max():.2f} us (span {ex.max():.2f} us); tiles {U.min()}-{U.max()}; "
              f"per-CTA busy {dur.min():.2f}/{np.median(dur):.2f}/{dur.max():.2f} us (min/median/max)")
        order = np.argsort(-ex)[:6]
        print("  slowest CTAs (id, tiles, exit us, busy us):",
              [(int(i), int(U[i]), round(float(ex[i]), 2), round(float(dur[i]), 2)) for i in order])
        for u in sorted(set(U.tolist())):
            m = U == u
            print(f"  tiles {u}: {m.sum()} CTAs, busy median {np.median(dur[m]):.2f} us, us/tile {np.median(dur[m]) / u:.3f}")
    t0 = t[0, 0, 0]
    if t0 == 0:
        print("no trace (CTA 0 ran no tiles, or not the tensor-core pass)")
        return
    rel = np.where(t > 0, t - t0, -1)
    print(f"{cfgname}: kernel entry 0, predecessor done {rel[0, 0, 4]}, end {rel[0, 0, 5]} cycles")
    hdr = ["u", "P", "X1", "X2", "G1s", "G1w", "G1c", "G2s", "G2w", "G2c", "STf", "STr", "Es", "Et", "Ed", "Ea", "Ec",
           "Eb", "Ee"]
    print(" ".join(f"{h:>6s}" for h in hdr))
    for u in range(256):
        if rel[0, u, 1] < 0:
            break
        wg = 3 + (u & 1)
        row = [u, rel[0, u, 1], rel[0, u, 2], rel[0, u, 3], rel[1, u, 0], rel[1, u, 1], rel[1, u, 2], rel[1, u, 3],
               rel[1, u, 4], rel[1, u, 5], rel[2, u, 1], rel[2, u, 2]] + [rel[wg, u, e] for e in range(7)]
        print(" ".join(f"{v:6d}" for v in row))


if __name__ == "__main__":
    main()
