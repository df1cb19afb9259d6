mkdir -p gpurun_out
timeout 900 python -m pytest -m gpu -q tests/test_gpu_parity.py -k "graph" > gpurun_out/pytest_new.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_new.log
