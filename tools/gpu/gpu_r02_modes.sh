# round 2: templated pass variants (plain / check / p2p-y), GEMM1 f16 vs tf32 at C3-C5, C4 K=1000 parity record
mkdir -p gpurun_out
python -c "import paper_1608_02227_b200.build as b; b.build()" > gpurun_out/build.log 2>&1
run() { t=$1; C=$2; S=$3; shift 3; env "$@" timeout 600 python bench.py --config $C --steps $S --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/m_${t}_${C}.json 2>&1; }
for C in C4 C5; do run f16 $C 20 X=0; run tf32 $C 20 CR_TC_G1_TF32=1; done
run f16 C3 2000 X=0; run tf32 C3 2000 CR_TC_G1_TF32=1
(cd _ab/ref && timeout 600 python bench.py --config C3 --steps 2000 --warmup 5 --no-cpu-baseline --no-e2e) > gpurun_out/m_ref_C3.json 2>&1
timeout 900 python tools/full_parity.py gpu C4 1000 > gpurun_out/full_parity_C4.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_tc_rings.py tests/test_gpu_p2p.py tests/test_gpu_nccl1.py -q -x > gpurun_out/pytest_modes.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_modes.log
