"""Per-instruction stall attribution of an ncu report, mapped to kernel source lines via nvdisasm -g.

    python tools/ncu_stalls.py gpurun_out/prof_C4.ncu-rep 40 [reason]            (pass_tc_kernel<40>)
    KERNEL=resident SRC=resident.cu FUNC='resident_kernelIfLi16E' python tools/ncu_stalls.py rep.ncu-rep x
"""
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, NK = sys.argv[1], sys.argv[2]
reason = sys.argv[3] if len(sys.argv) > 3 else "Warp Stall Sampling (All Samples)"
kf = ["-k", "regex:" + os.environ["KFILTER"]] if os.environ.get("KFILTER") else []
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"] + kf,
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, data = rows[1], rows[2:]
for _i, _r in enumerate(data):                      # several kernels: keep the first section
    if _r and _r[0] == "Kernel Name":
        data = data[:_i]
        break
ai, si, ri = h.index("Address"), h.index("Source"), h.index(reason)
base = int(data[0][ai], 16)
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
so = os.path.join(root, "paper_1608_02227_b200", "libcr.so")
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", so], cwd=d, capture_output=True)
KER = os.environ.get("KERNEL", "pass_tc")
SRCF = os.environ.get("SRC", "pass_tc.cu")
FUNC = os.environ.get("FUNC", "pass_tc_kernelILi%sE" % NK)
dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, KER + ".sm_100a.cubin")], capture_output=True,
                     text=True).stdout.split("\n")
start = [i for i, l in enumerate(dis) if re.match(r"\s*\.text\._ZN.*%s" % FUNC, l)][0]
line_of, last = {}, None
for l in dis[start + 1:]:
    if re.match(r"\s*\.text\.", l):
        break
    m = re.search(r'//## File ".*%s", line (\d+)' % re.escape(SRCF), l)
    if m:
        last = int(m.group(1))
    mo = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if mo:
        line_of[int(mo.group(1), 16)] = last
src = open(os.path.join(root, "paper_1608_02227_b200", "csrc", "kernels", SRCF)).read().split("\n")
agg = {}
tot = 0.0
for r in data:
    try:
        v = float(r[ri] or 0)
    except ValueError:
        continue
    tot += v
    ln = line_of.get(int(r[ai], 16) - base)
    agg[ln] = agg.get(ln, 0.0) + v
print(f"{reason}: total {tot:.0f}; by last {SRCF} line at or before the instruction")
for ln, v in sorted(agg.items(), key=lambda t: -t[1])[:25]:
    print(f"{100 * v / tot:6.1f}%  L{ln}: {src[ln - 1].strip()[:90] if ln else ''}")
