mkdir -p gpurun_out
timeout 900 python -m pytest -m gpu -q -x tests/test_gpu_parity.py -k "lipschitz or smoke or C1 or C2_500" > gpurun_out/pytest_new.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_new.log
for c in "C4 1000" "C5 200" "C3 2000"; do python tools/e2e_breakdown.py $c >> gpurun_out/e2e.txt 2>&1; HOST_L=1 python tools/e2e_breakdown.py $c >> gpurun_out/e2e.txt 2>&1; done
