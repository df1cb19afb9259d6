mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/smi.txt 2>&1
python -c "import paper_1608_02227_b200.build as b; b.build()" > gpurun_out/build.log 2>&1
timeout 300 python tools/primal_probe.py C4 5 > gpurun_out/primal_C4.txt 2>&1
CUDA_MODULE_LOADING=EAGER timeout 300 python tools/primal_probe.py C4 5 >> gpurun_out/primal_C4.txt 2>&1
timeout 300 python tools/primal_probe.py C5 3 > gpurun_out/primal_C5.txt 2>&1
timeout 600 python bench.py --config C5 --steps 20 --warmup 5 > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err
timeout 600 python bench.py --config C4 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
