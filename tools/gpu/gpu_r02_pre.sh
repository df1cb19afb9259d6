# round 2: Theta / X loads issued before the programmatic-dependency wait; smoke; residual ncu; init profile
mkdir -p gpurun_out
python -c "import paper_1608_02227_b200.build as b; b.build()" > gpurun_out/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
run() { t=$1; C=$2; S=$3; shift 3; env "$@" timeout 600 python bench.py --config $C --steps $S --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/p_${t}_${C}.json 2>&1; }
run pre C3 2000 X=0; run pre C4 20 X=0; run pre C5 20 X=0
(cd _ab/ref && timeout 600 python bench.py --config C3 --steps 2000 --warmup 5 --no-cpu-baseline --no-e2e) > gpurun_out/p_ref_C3.json 2>&1
CR_INIT_PROF=1 timeout 300 python tools/primal_probe.py C5 2 > gpurun_out/initprof_C5.txt 2>&1
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tc_rings.py tests/test_gpu_p2p.py tests/test_gpu_nccl1.py tests/test_gpu_adaptive.py -q -x -k "not full_size and not C3_full" > gpurun_out/pytest_pre.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_pre.log
timeout 300 python tools/primal_once.py C5 > gpurun_out/primal_once.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:residual2 -c 1 -o gpurun_out/res_C5 python tools/primal_once.py C5 > gpurun_out/ncu_res.log 2>&1
