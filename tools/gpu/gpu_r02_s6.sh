# round 2, session 4: the tree with the zero-tile GEMM2 skip -- smoke, full GPU suite, default bench lines
mkdir -p gpurun_out/s6
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s6/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s6/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/s6/smoke.log
timeout 900 python bench.py > gpurun_out/s6/bench_C5.json 2> gpurun_out/s6/bench_C5.err
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/s6/bench_C5_driverargs.json 2> gpurun_out/s6/bench_C5_driverargs.err
timeout 900 python bench.py --config C4 > gpurun_out/s6/bench_C4.json 2> gpurun_out/s6/bench_C4.err
timeout 900 python bench.py --config C4 --steps 20 --warmup 5 > gpurun_out/s6/bench_C4_driverargs.json 2> gpurun_out/s6/bench_C4_driverargs.err
timeout 900 python bench.py --config C3 > gpurun_out/s6/bench_C3.json 2> gpurun_out/s6/bench_C3.err
timeout 2700 python -m pytest tests -m gpu -q > gpurun_out/s6/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s6/pytest_gpu.log
