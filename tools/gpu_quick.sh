mkdir -p gpurun_out
python tools/resident_trace.py C2 > gpurun_out/rtrace.txt 2>&1; python tools/resident_trace.py C1 >> gpurun_out/rtrace.txt 2>&1
timeout 900 python -m pytest -m gpu -q -x tests/test_gpu_resident.py tests/test_gpu_parity.py -k "resident or C1 or C2 or smoke or single_step_fp64" > gpurun_out/pytest_new.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_new.log
b() { tag=$1; shift; env "$@" timeout 300 python bench.py --no-cpu-baseline --no-e2e $CFG > gpurun_out/q_$tag.json 2> gpurun_out/q_$tag.err; }
CFG="--config C2"; b C2 X=1
CFG="--config C1"; b C1 X=1
