# round 2, session 4: new = e9 (adaptive sums compiled out of the plain variant) + TC_TRACE compiled out of
# production builds, vs e9 (_ab/e9); trace build check (tools/tc_trace.py needs -DCR_TC_TRACE_BUILD)
mkdir -p gpurun_out/e14
for C in C4 C5 C3; do
  A="--config $C --steps 20 --warmup 10 --no-e2e --no-cpu-baseline"
  [ $C = C3 ] && A="--config $C --steps 400 --warmup 20 --no-e2e --no-cpu-baseline"
  for rep in 1 2 3; do
    timeout 600 python bench.py $A > gpurun_out/e14/new_${C}_$rep.json 2>/dev/null
    (cd _ab/e9 && timeout 600 python bench.py $A) > gpurun_out/e14/e9_${C}_$rep.json 2>/dev/null
  done
done
