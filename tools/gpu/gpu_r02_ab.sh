# round 2: A/B of the tcgen05 pass variants (GEMM1 f16 vs tf32) at C3/C4/C5 after the check-macro fix
mkdir -p gpurun_out
python -c "import paper_1608_02227_b200.build as b; b.build()" > gpurun_out/build.log 2>&1
for C in C4 C5 C3; do
  S=20; [ $C = C3 ] && S=2000
  timeout 600 python bench.py --config $C --steps $S --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab_${C}_f16.json 2>&1
  CR_TC_G1_TF32=1 timeout 600 python bench.py --config $C --steps $S --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab_${C}_tf32.json 2>&1
done
timeout 600 python bench.py --config C5 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab_C5_f16_b.json 2>&1
timeout 900 python -m pytest tests/test_gpu_p2p.py tests/test_gpu_nccl1.py tests/test_gpu_tc_rings.py -q -x > gpurun_out/pytest_p2p.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_p2p.log
