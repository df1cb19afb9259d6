mkdir -p gpurun_out
for a in "2400 20 quad" "2400 20 exp" "2400 80 quad" "2400 80 exp" "1600 20 quad"; do timeout 900 python tools/paper_workload.py $a 40000 >> gpurun_out/paper_wl.txt 2>&1; done
