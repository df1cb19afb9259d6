# round 2: bench lines C1-C5 (default = C5 with e2e and cpu_baseline), launch lists and one ncu --set full
# capture of the fused pass at C5 and C4 (each after the same command exited 0 without ncu)
mkdir -p gpurun_out/final
python -c "import paper_1608_02227_b200.build as b; b.build()" > gpurun_out/final/build.log 2>&1
timeout 900 python bench.py > gpurun_out/final/bench_C5.json 2> gpurun_out/final/bench_C5.err
for C in C4 C3 C2 C1; do timeout 900 python bench.py --config $C > gpurun_out/final/bench_$C.json 2> gpurun_out/final/bench_$C.err; done
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/final/bench_C5_driverargs.json 2> gpurun_out/final/bench_C5_driverargs.err
for C in C5 C4; do
  A="--config $C --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
  timeout 600 python bench.py $A > gpurun_out/final/plain_$C.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final/launches_$C.csv python bench.py $A > gpurun_out/final/ncu_launch_$C.log 2>&1
  timeout 600 python bench.py $A > gpurun_out/final/plain2_$C.log 2>&1 && \
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:pass_tc -s 4 -c 1 -o gpurun_out/final/prof_$C python bench.py $A > gpurun_out/final/ncu_full_$C.log 2>&1
done
