# round 2: GEMM2 in kind::f16 (bound-scaled Theta^k) for the F16 pass variant -- parity + C5 rate
mkdir -p gpurun_out
python -c "import paper_1608_02227_b200.build as b; b.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -s -k "tensor_core or edge_shapes or data_scale or pass_sums or C2_config or stats_against" > gpurun_out/pytest_g2f16.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_g2f16.log
timeout 600 python bench.py --config C5 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/g2f16_C5.json 2>&1
CR_TC_G1_TF32=1 timeout 600 python bench.py --config C5 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/g2f16_C5_tf32.json 2>&1
timeout 600 python bench.py --config C5 --steps 200 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/g2f16_C5_200.json 2>&1
