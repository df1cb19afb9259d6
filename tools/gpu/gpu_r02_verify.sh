# round 2: verify residual pass v2, fused reduce+prologue, graph prebuild, bench changes
mkdir -p gpurun_out
python -c "import paper_1608_02227_b200.build as b; b.build()" > gpurun_out/build.log 2>&1
timeout 300 python tools/primal_probe.py C4 5 > gpurun_out/primal_C4.txt 2>&1
timeout 300 python tools/primal_probe.py C5 3 > gpurun_out/primal_C5.txt 2>&1
timeout 300 python tools/primal_probe.py C3 5 > gpurun_out/primal_C3.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "not full_size and not C3_full" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --config C4 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err
timeout 600 python bench.py --config C3 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_C3.json 2> gpurun_out/bench_C3.err
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err
timeout 900 bash tools/tc_sweep_c5.sh C5 > gpurun_out/sweep_C5.txt 2>&1
