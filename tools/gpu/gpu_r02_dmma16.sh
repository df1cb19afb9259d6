# round 2: residual pass with mma.m16n8k4 f64 -- parity of the diagnostics + primal timings
mkdir -p gpurun_out
python -c "import paper_1608_02227_b200.build as b; b.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "stats_against or K_iterations_C1 or K_iterations_C2_500 or K_iterations_C3_reduced or constant_ybar" > gpurun_out/pytest_dmma16.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_dmma16.log
for C in C4 C5 C3; do timeout 300 python tools/primal_probe.py $C 3 > gpurun_out/dmma16_$C.txt 2>&1; done
