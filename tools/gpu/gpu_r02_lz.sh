# round 2: device Lanczos start vector, residual KC=16 / 2 stages; parity subset; primal + init timings; bench
mkdir -p gpurun_out
python -c "import paper_1608_02227_b200.build as b; b.build()" > gpurun_out/build.log 2>&1
CR_INIT_PROF=1 timeout 300 python tools/primal_probe.py C5 3 > gpurun_out/initprof_C5.txt 2>&1
CR_INIT_PROF=1 timeout 300 python tools/primal_probe.py C4 5 > gpurun_out/initprof_C4.txt 2>&1
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_continuation.py tests/test_abi.py -q -x -k "not full_size and not C3_full" > gpurun_out/pytest_lz.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_lz.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/lz_C5.json 2> gpurun_out/lz_C5.err
timeout 900 python bench.py --config C4 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/lz_C4.json 2> gpurun_out/lz_C4.err
