mkdir -p gpurun_out
timeout 900 python -m pytest -m gpu -q -x tests/test_gpu_adaptive.py tests/test_gpu_continuation.py tests/test_gpu_sharded_local.py > gpurun_out/pytest_new.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_new.log
b() { tag=$1; shift; env "$@" timeout 300 python bench.py --no-cpu-baseline --no-e2e $CFG > gpurun_out/q_$tag.json 2> gpurun_out/q_$tag.err; }
CFG="--config C4 --steps 200 --step adaptive"; b C4_ad X=1
CFG="--config C2 --steps 500 --step adaptive"; b C2_ad X=1
