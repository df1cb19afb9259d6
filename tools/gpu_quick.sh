mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
b() { tag=$1; shift; env "$@" timeout 300 python bench.py --no-cpu-baseline --no-e2e $CFG > gpurun_out/q_$tag.json 2> gpurun_out/q_$tag.err; }
CFG="--config C4"; b C4 X=1; b C4_3 CR_TC_STAGES=3; b C4_5 CR_TC_STAGES=5 CR_TC_G1STAGES=2 CR_TC_G2STAGES=2
CFG="--config C5 --steps 40"; b C5 X=1; b C5_3 CR_TC_STAGES=3 CR_TC_G1STAGES=3 CR_TC_G2STAGES=2
CFG="--config C3"; b C3 X=1; b C3_3 CR_TC_STAGES=3
