# round 2, session 7 (restored container): rebuild, smoke, default bench line (C5) and C4 with the
# driver's args, to confirm the restored tree on a fresh box
mkdir -p gpurun_out/s7
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s7/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s7/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/s7/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/s7/bench_C5_driverargs.json 2> gpurun_out/s7/bench_C5_driverargs.err
timeout 900 python bench.py --config C4 --steps 20 --warmup 5 > gpurun_out/s7/bench_C4_driverargs.json 2> gpurun_out/s7/bench_C4_driverargs.err
timeout 900 python -m pytest tests -m gpu -q -x -k "parity or abi" > gpurun_out/s7/pytest_gpu_parity.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s7/pytest_gpu_parity.log
