# round 2: three epilogue warpgroups (NWG=3) -- same-box rate A/B vs NWG=2, then parity + ring stress
mkdir -p gpurun_out
python -c "import paper_1608_02227_b200.build as b; b.build()" > gpurun_out/build.log 2>&1
run() { t=$1; C=$2; S=$3; shift 3; env "$@" timeout 600 python bench.py --config $C --steps $S --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/nwg_${t}_${C}.json 2>&1; }
for C in C5 C4; do run w3 $C 20 X=0; run w2 $C 20 CR_TC_NWG=2; run w3b $C 20 X=0; run w2b $C 20 CR_TC_NWG=2; done
run w3 C3 2000 X=0; run w2 C3 2000 CR_TC_NWG=2
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tc_rings.py tests/test_gpu_adaptive.py tests/test_gpu_partition.py -q -x -k "not full_size" > gpurun_out/pytest_nwg.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_nwg.log
