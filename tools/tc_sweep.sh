#!/bin/bash
# Sweep the tcgen05 pass's knobs at one config (one line per setting): ring depths, producer
# back-off, L2 policy for Theta.  Usage: bash tools/tc_sweep.sh C4
C=${1:-C4}
run() { echo -n "$* : "; env "$@" python bench.py --config $C --no-cpu-baseline --no-e2e --steps 300 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],5), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])"; }
run X=0
run CR_TC_STAGES=4
run CR_TC_STAGES=6 CR_TC_G1STAGES=2 CR_TC_G2STAGES=2
run CR_TC_G1STAGES=2 CR_TC_G2STAGES=3
run CR_TC_POLL_NS=0
run CR_TC_POLL_NS=256
run CR_TC_THETA_L2=0
run CR_TC_THETA_L2=1
run CR_NO_PDL=1
run X=0
