# round 2: after reverting the 3-warpgroup experiment -- rings (run-ahead forces even depths), parity subset, rates
mkdir -p gpurun_out
python -c "import paper_1608_02227_b200.build as b; b.build()" > gpurun_out/build.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_tc_rings.py tests/test_gpu_parity.py -q -x -k "not full_size and not C3_full" > gpurun_out/pytest_post.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_post.log
for C in C5 C4; do timeout 600 python bench.py --config $C --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/post_$C.json 2>&1; done
timeout 600 python bench.py --config C3 --steps 2000 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/post_C3.json 2>&1
