# round 2, session 4: Theta loads before the PDL wait (CR_TC_PREWAIT) and evict-last Theta^k stores
# (CR_TC_THETA_L2 bit 2) vs the RED-flush commit (_ab/r1)
mkdir -p gpurun_out/pre
B="--steps 400 --warmup 20 --no-e2e --no-cpu-baseline"
for rep in 1 2; do
  (cd _ab/r1 && timeout 600 python bench.py --config C3 $B) > gpurun_out/pre/r1_C3_$rep.json 2>/dev/null
  timeout 600 python bench.py --config C3 $B > gpurun_out/pre/new0_C3_$rep.json 2>/dev/null
  CR_TC_PREWAIT=1 timeout 600 python bench.py --config C3 $B > gpurun_out/pre/new1_C3_$rep.json 2>/dev/null
  for L in 1 3 4 5; do
    CR_TC_PREWAIT=1 CR_TC_THETA_L2=$L timeout 600 python bench.py --config C3 $B > gpurun_out/pre/new1_l2$L\_C3_$rep.json 2>/dev/null
  done
done
A="--config C4 --steps 20 --warmup 10 --no-e2e --no-cpu-baseline"
for rep in 1 2; do
  (cd _ab/r1 && timeout 600 python bench.py $A) > gpurun_out/pre/r1_C4_$rep.json 2>/dev/null
  timeout 600 python bench.py $A > gpurun_out/pre/new0_C4_$rep.json 2>/dev/null
  CR_TC_PREWAIT=1 timeout 600 python bench.py $A > gpurun_out/pre/new1_C4_$rep.json 2>/dev/null
done
