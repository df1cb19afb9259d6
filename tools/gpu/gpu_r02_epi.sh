# round 2, session 4: epilogue variants vs the RED-flush commit (_ab/r1):
#   new  = 4-chain column sums;  m = new + both S' halves loaded from TMEM at once;
# and the fp64 SIMT pass with one CTA per SM (new) vs two (r1)
mkdir -p gpurun_out/epi
for C in C4 C5 C3; do
  A="--config $C --steps 20 --warmup 10 --no-e2e --no-cpu-baseline"
  [ $C = C3 ] && A="--config $C --steps 400 --warmup 20 --no-e2e --no-cpu-baseline"
  for rep in 1 2; do
    (cd _ab/r1 && timeout 600 python bench.py $A) > gpurun_out/epi/r1_${C}_$rep.json 2>/dev/null
    timeout 600 python bench.py $A > gpurun_out/epi/new_${C}_$rep.json 2>/dev/null
    (cd _ab/m && timeout 600 python bench.py $A) > gpurun_out/epi/m_${C}_$rep.json 2>/dev/null
  done
done
(cd _ab/r1 && timeout 300 python tools/simt64_time.py 4000 20 50) > gpurun_out/epi/simt64_r1.txt 2>&1
timeout 300 python tools/simt64_time.py 4000 20 50 > gpurun_out/epi/simt64_new.txt 2>&1
(cd _ab/r1 && timeout 300 python tools/simt64_time.py 4000 8 50) >> gpurun_out/epi/simt64_r1.txt 2>&1
timeout 300 python tools/simt64_time.py 4000 8 50 >> gpurun_out/epi/simt64_new.txt 2>&1
