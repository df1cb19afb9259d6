# round 2, session 4: fp64 Theta X running sum in TMEM without the epilogue sub-phase events (new) vs the
# coalesced-flush commit (_ab/ref); sub-phase timelines from a -DCR_TC_SUBTRACE build (_ab/sub)
mkdir -p gpurun_out/acc2
(cd _ab/sub && CR_TC_TRACE_U0=200 timeout 300 python tools/tc_trace.py C4 30) > gpurun_out/acc2/trace_C4_200_sub.txt 2>&1
CR_TC_TRACE_U0=200 timeout 300 python tools/tc_trace.py C4 30 > gpurun_out/acc2/trace_C4_200.txt 2>&1
for C in C4 C3 C5; do
  A="--config $C --steps 20 --warmup 10 --no-e2e --no-cpu-baseline"
  [ $C = C3 ] && A="--config $C --steps 400 --warmup 20 --no-e2e --no-cpu-baseline"
  for rep in 1 2; do
    timeout 600 python bench.py $A > gpurun_out/acc2/new_${C}_$rep.json 2> gpurun_out/acc2/new_${C}_$rep.err
    (cd _ab/ref && timeout 600 python bench.py $A) > gpurun_out/acc2/ref_${C}_$rep.json 2> gpurun_out/acc2/ref_${C}_$rep.err
  done
done
