# round 2, session 4: fp64 Theta X running sum in TMEM (new) vs the coalesced-flush commit (_ab/ref)
mkdir -p gpurun_out/acc
CR_TC_TRACE_U0=3500 timeout 600 python tools/tc_trace.py C5 30 > gpurun_out/acc/trace_C5_3500.txt 2>&1
CR_TC_TRACE_U0=200 timeout 300 python tools/tc_trace.py C4 30 > gpurun_out/acc/trace_C4_200.txt 2>&1
for C in C5 C4 C3; do
  A="--config $C --steps 20 --warmup 10 --no-e2e --no-cpu-baseline"
  [ $C = C3 ] && A="--config $C --steps 400 --warmup 20 --no-e2e --no-cpu-baseline"
  for rep in 1 2; do
    timeout 600 python bench.py $A > gpurun_out/acc/new_${C}_$rep.json 2> gpurun_out/acc/new_${C}_$rep.err
    (cd _ab/ref && timeout 600 python bench.py $A) > gpurun_out/acc/ref_${C}_$rep.json 2> gpurun_out/acc/ref_${C}_$rep.err
  done
done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tc_rings.py -q -x > gpurun_out/acc/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/acc/pytest.log
