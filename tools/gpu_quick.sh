mkdir -p gpurun_out
timeout 1200 python -m pytest -m gpu -q -x tests/test_gpu_parity.py -k "full_size" > gpurun_out/pytest_new.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_new.log
free -g >> gpurun_out/pytest_new.log; nproc >> gpurun_out/pytest_new.log
