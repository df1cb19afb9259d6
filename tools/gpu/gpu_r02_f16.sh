# round 2: kind::f16 GEMM1 (parity + bench), residual v3 (16 warps)
mkdir -p gpurun_out
python -c "import paper_1608_02227_b200.build as b; b.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -s -k "tensor_core or edge_shapes or data_scale or C2_config or pass_sums or stats_against" > gpurun_out/pytest_f16.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_f16.log
timeout 300 python tools/primal_probe.py C4 5 > gpurun_out/primal_C4.txt 2>&1
timeout 300 python tools/primal_probe.py C5 3 > gpurun_out/primal_C5.txt 2>&1
timeout 600 python bench.py --config C5 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_C5_f16.json 2> gpurun_out/bench_C5_f16.err
CR_TC_G1_TF32=1 timeout 600 python bench.py --config C5 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_C5_tf32.json 2> gpurun_out/bench_C5_tf32.err
timeout 600 python bench.py --config C4 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_C4_f16.json 2> gpurun_out/bench_C4_f16.err
timeout 600 python bench.py --config C3 --steps 2000 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_C3_f16.json 2> gpurun_out/bench_C3_f16.err
timeout 1800 python -m pytest tests/test_gpu_parity.py -q -x -s -k "full_size or C3_full" > gpurun_out/pytest_f16_full.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_f16_full.log
