# round 2: control run -- r01 kernels (commit d1fab78, built into _ab/ref) vs the current tree on the SAME box,
# plus a torch copy-bandwidth probe of the box
mkdir -p gpurun_out
python -c "import paper_1608_02227_b200.build as b; b.build()" > gpurun_out/build.log 2>&1
python tools/stream_roofline.py > gpurun_out/ctrl_stream.txt 2>&1
for C in C4 C5; do
  (cd _ab/ref && timeout 600 python bench.py --config $C --steps 20 --warmup 5 --no-cpu-baseline --no-e2e) > gpurun_out/ctrl_${C}_r01.json 2>&1
  timeout 600 python bench.py --config $C --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ctrl_${C}_now.json 2>&1
  CR_NO_FUSE=1 timeout 600 python bench.py --config $C --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ctrl_${C}_nofuse.json 2>&1
done
timeout 300 python tools/primal_probe.py C4 5 > gpurun_out/primal_C4.txt 2>&1
timeout 300 python tools/primal_probe.py C5 3 > gpurun_out/primal_C5.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "stats_against or K_iterations_C2_500 or K_iterations_C1 or K_iterations_C3_reduced or constant_ybar" > gpurun_out/pytest_res.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_res.log
