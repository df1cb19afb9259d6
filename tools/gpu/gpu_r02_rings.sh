# round 2: ring-protocol stress (depths 2-6, GEMM1 run-ahead, in-kernel checks), primal launch list
mkdir -p gpurun_out
python -c "import paper_1608_02227_b200.build as b; b.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_tc_rings.py -q -rA > gpurun_out/pytest_rings.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_rings.log
for R in 0 1; do CR_TC_G1_RUNAHEAD=$R timeout 600 python bench.py --config C5 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_C5_ra$R.json 2>&1; done
CR_TC_G1_RUNAHEAD=1 timeout 600 python bench.py --config C4 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_C4_ra1.json 2>&1
timeout 300 python tools/primal_once.py C4 > gpurun_out/primal_once.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_primal_C4.csv -k regex:"residual|transpose|stats_finalize|prologue" python tools/primal_once.py C4 > gpurun_out/ncu_primal.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_primal_C5.csv -k regex:"residual|transpose|stats_finalize|prologue" python tools/primal_once.py C5 >> gpurun_out/ncu_primal.log 2>&1
