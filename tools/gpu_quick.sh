mkdir -p gpurun_out
timeout 900 python -m pytest -m gpu -q -x tests/test_gpu_continuation.py tests/test_gpu_adaptive.py > gpurun_out/pytest_new.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_new.log
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/q_C4.json 2> gpurun_out/q_C4.err
