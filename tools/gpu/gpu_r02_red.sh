# round 2, session 4: Theta X window flush by fp64 RED (r1: HEAD + RED; new: + trace records) vs HEAD (_ab/ref)
mkdir -p gpurun_out/red
for C in C4 C3 C5; do
  A="--config $C --steps 20 --warmup 10 --no-e2e --no-cpu-baseline"
  [ $C = C3 ] && A="--config $C --steps 400 --warmup 20 --no-e2e --no-cpu-baseline"
  for rep in 1 2; do
    timeout 600 python bench.py $A > gpurun_out/red/new_${C}_$rep.json 2> gpurun_out/red/new_${C}_$rep.err
    (cd _ab/r1 && timeout 600 python bench.py $A) > gpurun_out/red/r1_${C}_$rep.json 2> gpurun_out/red/r1_${C}_$rep.err
    (cd _ab/ref && timeout 600 python bench.py $A) > gpurun_out/red/ref_${C}_$rep.json 2> gpurun_out/red/ref_${C}_$rep.err
  done
done
CR_TC_TRACE_U0=3500 timeout 600 python tools/tc_trace.py C5 30 > gpurun_out/red/trace_C5_3500.txt 2>&1
