# round 2: GEMM1 2-pass option at C5 / C4 (bench + parity), primal timing, full gpu suite
mkdir -p gpurun_out
python -c "import paper_1608_02227_b200.build as b; b.build()" > gpurun_out/build.log 2>&1
timeout 300 python tools/primal_probe.py C4 5 > gpurun_out/primal_C4.txt 2>&1
timeout 300 python tools/primal_probe.py C5 3 > gpurun_out/primal_C5.txt 2>&1
for P in 3 2; do
  CR_TC_G1PASSES=$P timeout 600 python bench.py --config C5 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_C5_p$P.json 2> gpurun_out/bench_C5_p$P.err
  CR_TC_G1PASSES=$P timeout 600 python bench.py --config C4 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_C4_p$P.json 2> gpurun_out/bench_C4_p$P.err
done
CR_TC_G1PASSES=2 timeout 1800 python -m pytest tests/test_gpu_parity.py -x -q -s -k "tensor_core or edge_shapes or C3_full or full_size or C2_config or pass_sums" > gpurun_out/pytest_p2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_p2.log
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
