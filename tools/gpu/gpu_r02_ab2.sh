# round 2: locate the tcgen05-pass regression -- r01 kernels vs the current tree with features compiled out
mkdir -p gpurun_out
python -c "import paper_1608_02227_b200.build as b; b.build()" > gpurun_out/build.log 2>&1
run() {  # dir tag config env...
  d=$1; t=$2; C=$3; shift 3
  (cd $d && env "$@" timeout 600 python bench.py --config $C --steps 20 --warmup 5 --no-cpu-baseline --no-e2e) > gpurun_out/ab2_${t}_${C}.json 2>&1
}
for C in C4 C5; do
  run _ab/ref ref $C X=0
  run . cur_f16 $C X=0
  run . cur_tf32 $C CR_TC_G1_TF32=1
  run _ab/nochk nochk_f16 $C X=0
  run _ab/nochk_nop2p nochk_nop2p_f16 $C X=0
  run _ab/nochk_nop2p nochk_nop2p_tf32 $C CR_TC_G1_TF32=1
  run _ab/ref ref2 $C X=0
done
