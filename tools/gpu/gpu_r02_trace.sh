mkdir -p gpurun_out/t1
for C in C3 C4 C5; do timeout 300 python tools/tc_trace.py $C 12 > gpurun_out/t1/trace_$C.txt 2>&1; done
timeout 300 python bench.py --config C3 --steps 200 --warmup 20 --no-e2e --no-cpu-baseline > gpurun_out/t1/bench_C3.json 2> gpurun_out/t1/bench_C3.err
