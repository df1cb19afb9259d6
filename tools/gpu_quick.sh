mkdir -p gpurun_out
b() { tag=$1; shift; env "$@" timeout 300 python bench.py --no-cpu-baseline --no-e2e $CFG > gpurun_out/q_$tag.json 2> gpurun_out/q_$tag.err; }
CFG="--config C4"; b C4_532 X=1; b C4_433 CR_TC_STAGES=4; b C4_522 CR_TC_G1STAGES=2 CR_TC_G2STAGES=2; b C4_333 CR_TC_STAGES=3; b C4_532b X=1; b C4_444 CR_TC_STAGES=4 CR_TC_G1STAGES=4 CR_TC_G2STAGES=4
