#!/bin/bash
# C5 ring-depth sweep of the tcgen05 pass (GEMM1 in kind::f16: X_J slots of 10 KB, X_J^T slots of
# 20 KB, Theta slots of 32 KB, 227 KB of shared memory); 20 timed iterations after 5 warm-up,
# as the driver runs bench.py.  Usage: bash tools/tc_sweep_c5.sh [C5]
C=${1:-C5}
run() { echo -n "$* : "; env "$@" python bench.py --config $C --no-cpu-baseline --no-e2e --steps 20 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],5), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; }
run X=0
run CR_TC_STAGES=6 CR_TC_G1STAGES=1 CR_TC_G2STAGES=1
run CR_TC_STAGES=5 CR_TC_G1STAGES=3 CR_TC_G2STAGES=1
run CR_TC_STAGES=5 CR_TC_G1STAGES=1 CR_TC_G2STAGES=2
run CR_TC_STAGES=4 CR_TC_G1STAGES=3 CR_TC_G2STAGES=3
run X=0
