# round 2, session 4: z = GEMM2 MMAs skipped for all-zero Theta^k tiles (exact) vs the final tree (new);
# C5 / C4 at full K (late iterations: 10-34% of tiles all zero) and K = 20; parity + ring tests on z
mkdir -p gpurun_out/z
for rep in 1 2; do
  for C in C5 C4; do
    A="--config $C --no-e2e --no-cpu-baseline"
    timeout 600 python bench.py $A > gpurun_out/z/new_${C}_$rep.json 2>/dev/null
    (cd _ab/z && timeout 600 python bench.py $A) > gpurun_out/z/z_${C}_$rep.json 2>/dev/null
  done
  A="--config C5 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline"
  timeout 600 python bench.py $A > gpurun_out/z/new_C5k20_$rep.json 2>/dev/null
  (cd _ab/z && timeout 600 python bench.py $A) > gpurun_out/z/z_C5k20_$rep.json 2>/dev/null
done
(cd _ab/z && timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tc_rings.py -q -x) > gpurun_out/z/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/z/pytest.log
