# round 2: C5 K=100 full-size parity record (the fp64 oracle needs ~22 s per C5 iteration on the box's 16
# cores: K=200 (~80 min) does not fit one 60-minute gpurun call, K=100 (~40 min) does)
mkdir -p gpurun_out
python -c "import paper_1608_02227_b200.build as b; b.build()" > gpurun_out/build.log 2>&1
timeout 3300 python tools/full_parity.py both C5 100 > gpurun_out/full_parity_C5.log 2>&1
