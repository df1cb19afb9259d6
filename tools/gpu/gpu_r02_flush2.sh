# round 2, session 4: coalesced Theta X flush + batched Xi' max (new) vs HEAD (_ab/ref; its lines from gpu_r02_flush.sh)
mkdir -p gpurun_out/fl
for C in C3 C4 C5; do timeout 300 python tools/tc_trace.py $C 12 > gpurun_out/fl/trace_$C.txt 2>&1; done
for C in C5 C4 C3; do
  A="--config $C --steps 20 --warmup 10 --no-e2e --no-cpu-baseline"
  [ $C = C3 ] && A="--config $C --steps 400 --warmup 20 --no-e2e --no-cpu-baseline"
  for rep in 1 2; do
    timeout 600 python bench.py $A > gpurun_out/fl/new_${C}_$rep.json 2> gpurun_out/fl/new_${C}_$rep.err
    (cd _ab/ref && timeout 600 python bench.py $A) > gpurun_out/fl/ref_${C}_$rep.json 2> gpurun_out/fl/ref_${C}_$rep.err
  done
done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tc_rings.py -q -x > gpurun_out/fl/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/fl/pytest.log
