# round 2, session 4: e9 = adaptive sums compiled out of the plain pass variant; e10 = e9 + rowscale hoisted
# + colpart written by the warps in turn; new = committed (4-chain column sums); parity subset on new
mkdir -p gpurun_out/e9
for C in C4 C5 C3; do
  A="--config $C --steps 20 --warmup 10 --no-e2e --no-cpu-baseline"
  [ $C = C3 ] && A="--config $C --steps 400 --warmup 20 --no-e2e --no-cpu-baseline"
  for rep in 1 2; do
    timeout 600 python bench.py $A > gpurun_out/e9/new_${C}_$rep.json 2>/dev/null
    (cd _ab/e9 && timeout 600 python bench.py $A) > gpurun_out/e9/e9_${C}_$rep.json 2>/dev/null
    (cd _ab/e10 && timeout 600 python bench.py $A) > gpurun_out/e9/e10_${C}_$rep.json 2>/dev/null
  done
done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tc_rings.py tests/test_gpu_adaptive.py -q -x > gpurun_out/e9/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/e9/pytest.log
