mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
b() { tag=$1; shift; env "$@" timeout 300 python bench.py --no-cpu-baseline --no-e2e $CFG > gpurun_out/q_$tag.json 2> gpurun_out/q_$tag.err; }
CFG="--config C3"; b C3_pdl X=1; b C3_nopdl CR_NO_PDL=1; b C3_pdl2 X=1
CFG="--config C4"; b C4_pdl X=1; b C4_nopdl CR_NO_PDL=1
