# round 2, session 3: re-validate the checkpointed tree (build as the driver does, smoke, GPU suite, default bench)
mkdir -p gpurun_out/s3pre
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s3pre/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3pre/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/s3pre/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/s3pre/bench_C5_driverargs.json 2> gpurun_out/s3pre/bench_C5_driverargs.err
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/s3pre/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s3pre/pytest_gpu.log
