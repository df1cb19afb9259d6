#!/bin/bash
# One GPU session: parity tests, smoke, bench lines per config (+ adaptive, partition), launch list.
# Copy the JSON lines into profiles/rNN/ afterwards (tools/show.py prints a summary).
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err
for c in C3 C5 C2 C1; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 600 python bench.py --step adaptive --config C4 --no-cpu-baseline > gpurun_out/bench_C4_adaptive.json 2> gpurun_out/bench_C4_adaptive.err
timeout 600 python bench.py --config C3 --nbar 100 --steps 100 --no-e2e > gpurun_out/bench_C3_nbar100.json 2> gpurun_out/bench_C3_nbar100.err
timeout 600 python bench.py --config C4 --nbar 64 --steps 50 --no-e2e > gpurun_out/bench_C4_nbar64.json 2> gpurun_out/bench_C4_nbar64.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_C4.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
