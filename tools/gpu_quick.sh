mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
t() { echo "== $*" >> gpurun_out/s3.txt; env "$@" timeout 200 python tools/probe/s3.py $ARGS >> gpurun_out/s3.txt 2>&1; }
ARGS="C4 3000 1"; t CR_TC_STAGES=3; t CR_TC_STAGES=2
ARGS="C5 200 1"; t CR_TC_STAGES=3
b() { tag=$1; shift; env "$@" timeout 300 python bench.py --no-cpu-baseline --no-e2e $CFG > gpurun_out/q_$tag.json 2> gpurun_out/q_$tag.err; }
CFG="--config C5 --steps 40"; b C5_4_2_2 CR_TC_STAGES=4 CR_TC_G1STAGES=2 CR_TC_G2STAGES=2; b C5_3_3_3 CR_TC_STAGES=3 CR_TC_G1STAGES=3 CR_TC_G2STAGES=3; b C5_3_3_2 CR_TC_STAGES=3 CR_TC_G1STAGES=3 CR_TC_G2STAGES=2; b C5_3_2_3 CR_TC_STAGES=3 CR_TC_G1STAGES=2 CR_TC_G2STAGES=3
CFG="--config C4"; b C4_4_3_3 CR_TC_STAGES=4; b C4_4_2_2 CR_TC_STAGES=4 CR_TC_G1STAGES=2 CR_TC_G2STAGES=2; b C4_3_3_3 CR_TC_STAGES=3; b C4_4_4_4 CR_TC_STAGES=4 CR_TC_G1STAGES=4 CR_TC_G2STAGES=4
for c in C4 C5; do timeout 120 python tools/tc_trace.py $c > gpurun_out/trace_$c.txt 2>&1; done
