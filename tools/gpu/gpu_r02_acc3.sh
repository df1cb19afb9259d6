# round 2, session 4: out-of-line flush with the TMEM running sum (new), out-of-line flush without it (_ab/x),
# the coalesced-flush commit (_ab/ref)
mkdir -p gpurun_out/acc3
for C in C4 C3; do
  A="--config $C --steps 20 --warmup 10 --no-e2e --no-cpu-baseline"
  [ $C = C3 ] && A="--config $C --steps 400 --warmup 20 --no-e2e --no-cpu-baseline"
  for rep in 1 2; do
    timeout 600 python bench.py $A > gpurun_out/acc3/new_${C}_$rep.json 2> gpurun_out/acc3/new_${C}_$rep.err
    (cd _ab/x && timeout 600 python bench.py $A) > gpurun_out/acc3/x_${C}_$rep.json 2> gpurun_out/acc3/x_${C}_$rep.err
    (cd _ab/ref && timeout 600 python bench.py $A) > gpurun_out/acc3/ref_${C}_$rep.json 2> gpurun_out/acc3/ref_${C}_$rep.err
  done
done
