# round 2 final: full GPU suite, smoke, bench lines (default C5 + C4/C3 with the driver's args and full K),
# launch lists reaching the fused pass
mkdir -p gpurun_out/final2
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/final2/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final2/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/final2/smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/final2/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final2/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/final2/bench_C5_driverargs.json 2> gpurun_out/final2/bench_C5_driverargs.err
timeout 900 python bench.py > gpurun_out/final2/bench_C5.json 2> gpurun_out/final2/bench_C5.err
timeout 900 python bench.py --config C4 --steps 20 --warmup 5 > gpurun_out/final2/bench_C4_driverargs.json 2> gpurun_out/final2/bench_C4_driverargs.err
timeout 900 python bench.py --config C4 > gpurun_out/final2/bench_C4.json 2> gpurun_out/final2/bench_C4.err
timeout 900 python bench.py --config C3 > gpurun_out/final2/bench_C3.json 2> gpurun_out/final2/bench_C3.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/final2/ref_C5.json 2> gpurun_out/final2/ref_C5.err
for C in C5 C4; do
  A="--config $C --steps 20 --warmup 5 --no-e2e --no-cpu-baseline"
  timeout 600 python bench.py $A > gpurun_out/final2/plain_$C.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/final2/launches_$C.csv python bench.py $A > gpurun_out/final2/ncu_$C.log 2>&1
done
