# round 2, session 4, final tree: build as the driver does, smoke, bench lines (default C5 + driver args,
# C4, C3), launch lists reaching the pass, one ncu --set full capture per config, full GPU suite
mkdir -p gpurun_out/s5
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s5/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s5/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/s5/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/s5/bench_C5_driverargs.json 2> gpurun_out/s5/bench_C5_driverargs.err
timeout 900 python bench.py > gpurun_out/s5/bench_C5.json 2> gpurun_out/s5/bench_C5.err
timeout 900 python bench.py --config C4 --steps 20 --warmup 5 > gpurun_out/s5/bench_C4_driverargs.json 2> gpurun_out/s5/bench_C4_driverargs.err
timeout 900 python bench.py --config C4 > gpurun_out/s5/bench_C4.json 2> gpurun_out/s5/bench_C4.err
timeout 900 python bench.py --config C3 > gpurun_out/s5/bench_C3.json 2> gpurun_out/s5/bench_C3.err
for C in C5 C4; do
  A="--config $C --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
  timeout 600 python bench.py $A > gpurun_out/s5/plain_$C.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/s5/launches_$C.csv python bench.py $A > gpurun_out/s5/ncu_launch_$C.log 2>&1
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:pass_tc -s 4 -c 1 -o gpurun_out/s5/prof_$C python bench.py $A > gpurun_out/s5/ncu_full_$C.log 2>&1
done
timeout 2700 python -m pytest tests -m gpu -q > gpurun_out/s5/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s5/pytest_gpu.log
