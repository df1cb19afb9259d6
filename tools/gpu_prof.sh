# ncu evidence for the fused pass: launch lists (C4, C5) and one --set full capture per config.
mkdir -p gpurun_out
CMD4="python bench.py --config C4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
CMD5="python bench.py --config C5 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD4 > gpurun_out/plain4.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_C4.csv $CMD4 > gpurun_out/ncu_l4.log 2>&1
$CMD5 > gpurun_out/plain5.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_C5.csv $CMD5 > gpurun_out/ncu_l5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:pass_tc -s 4 -c 1 -o gpurun_out/prof_C4 $CMD4 > gpurun_out/ncu_f4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:pass_tc -s 4 -c 1 -o gpurun_out/prof_C5 $CMD5 > gpurun_out/ncu_f5.log 2>&1
