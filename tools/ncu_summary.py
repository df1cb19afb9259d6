"""Summarise an ncu --set full report of the fused pass into profiles/ (text) and a traffic json.

    python tools/ncu_summary.py gpurun_out/prof_C4.ncu-rep C4 profiles/r01 "<command>"
"""
import csv
import io
import json
import os
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__grid_size",
        "launch__block_size"]
UNIT = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}


def main(rep, cfg, outdir, cmd, N=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u, v = rows[0], rows[1], rows[2]
    name = v[h.index("Kernel Name")] if "Kernel Name" in h else "?"
    lines = [f"# ncu --set full, {name[:60]}, {cfg}, 1 B200", f"# command: {cmd}",
             "# cold-cache serialized replay: compare shares / traffic, not absolute time"]
    for w in WANT:
        if w in h:
            i = h.index(w)
            lines.append(f"{w:75s} {v[i]:>14s} {u[i]}")
    stall = [(c, float(v[i])) for i, c in enumerate(h)
             if c.startswith("smsp__pcsamp_warps_issue_stalled_") and not c.endswith("_not_issued")
             and v[i].replace('.', '', 1).replace(',', '').isdigit()]
    tot = sum(x for _, x in stall) or 1.0
    lines.append("# warp stall samples (share)")
    for c, x in sorted(stall, key=lambda t: -t[1])[:8]:
        lines.append(f"  {100 * x / tot:6.1f}%  {c.replace('smsp__pcsamp_warps_issue_stalled_', '')}")
    rd = float(v[h.index("dram__bytes_read.sum")]) * UNIT[u[h.index("dram__bytes_read.sum")]]
    wr = float(v[h.index("dram__bytes_write.sum")]) * UNIT[u[h.index("dram__bytes_write.sum")]]
    if N:
        alg = 12.0 * N * N
        lines.append(f"# DRAM traffic per launch = {(rd + wr) / 1e9:.3f} GB vs algorithmic 12 B x N^2 = {alg / 1e9:.3f} GB"
                     f" ({(rd + wr) / alg:.3f}x)")
    os.makedirs(outdir, exist_ok=True)
    with open(os.path.join(outdir, f"{cfg}_pass_tc_ncu_full.txt"), "w") as f:
        f.write("\n".join(lines) + "\n")
    with open(os.path.join(os.path.dirname(outdir.rstrip("/")) or ".", f"traffic_{cfg}_tc.json"), "w") as f:
        json.dump({"bytes_per_launch": rd + wr, "source": os.path.join(outdir, f"{cfg}_pass_tc_ncu_full.txt"),
                   "kernel": name[:80], "config": cfg}, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4], int(sys.argv[5]) if len(sys.argv) > 5 else None)
