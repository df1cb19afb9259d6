# round 2: experiment -- GEMM2 in 2 passes (no Theta_lo X_hi): parity and C5 / C4 rate
mkdir -p gpurun_out
python -c "import paper_1608_02227_b200.build as b; b.build()" > gpurun_out/build.log 2>&1
CR_TC_G2PASSES=2 timeout 1200 python -m pytest tests/test_gpu_parity.py -q -s -k "tensor_core or edge_shapes or pass_sums or C2_config" > gpurun_out/pytest_g2p.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_g2p.log
CR_TC_G2PASSES=2 timeout 600 python bench.py --config C5 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/g2p_C5.json 2>&1
timeout 600 python bench.py --config C5 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/g3p_C5.json 2>&1
CR_TC_G2PASSES=2 timeout 1200 python -m pytest tests/test_gpu_parity.py -q -s -k "full_size_C5_beta" > gpurun_out/pytest_g2p_c5.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_g2p_c5.log
