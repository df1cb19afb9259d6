# round 2: residual pass v2b timing + ncu of one launch; full gpu suite
mkdir -p gpurun_out
python -c "import paper_1608_02227_b200.build as b; b.build()" > gpurun_out/build.log 2>&1
timeout 300 python tools/primal_probe.py C4 5 > gpurun_out/primal_C4.txt 2>&1
timeout 300 python tools/primal_probe.py C5 3 > gpurun_out/primal_C5.txt 2>&1
timeout 300 python tools/primal_once.py C4 > gpurun_out/primal_once.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:residual2 -c 1 -o gpurun_out/res_C4 python tools/primal_once.py C4 > gpurun_out/ncu_res.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
