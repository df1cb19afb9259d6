# round 2: full-size momentum tests extended to iteration 4 (checks GEMM2's Theta X at C4 / C5)
mkdir -p gpurun_out
python -c "import paper_1608_02227_b200.build as b; b.build()" > gpurun_out/build.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_parity.py -q -s -k "full_size" > gpurun_out/pytest_fs4.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_fs4.log
