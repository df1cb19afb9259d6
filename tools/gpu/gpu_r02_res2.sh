# round 2: residual pass with two CTAs per SM (128 x 64 tiles)
mkdir -p gpurun_out
python -c "import paper_1608_02227_b200.build as b; b.build()" > gpurun_out/build.log 2>&1
timeout 300 python tools/primal_probe.py C4 5 > gpurun_out/primal2_C4.txt 2>&1
timeout 300 python tools/primal_probe.py C5 3 > gpurun_out/primal2_C5.txt 2>&1
timeout 300 python tools/primal_probe.py C3 5 > gpurun_out/primal2_C3.txt 2>&1
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partition.py tests/test_gpu_sharded_local.py tests/test_gpu_continuation.py -q -x -k "not full_size" > gpurun_out/pytest_res2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_res2.log
