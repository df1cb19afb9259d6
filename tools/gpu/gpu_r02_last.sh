# round 2, last validation on the final tree: build as the driver does, smoke, full GPU suite, default bench line
mkdir -p gpurun_out/last
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/last/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/last/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/last/smoke.log
timeout 2700 python -m pytest tests -m gpu -q > gpurun_out/last/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/last/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/last/bench_C5_driverargs.json 2> gpurun_out/last/bench_C5_driverargs.err
timeout 900 python bench.py > gpurun_out/last/bench_C5.json 2> gpurun_out/last/bench_C5.err
