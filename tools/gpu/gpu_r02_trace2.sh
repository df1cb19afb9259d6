# round 2, session 4: C5 / C4 timelines at several points of the pass (CR_TC_TRACE_U0), effective clocks
mkdir -p gpurun_out/t2
for U0 in 0 3500 6800; do CR_TC_TRACE_U0=$U0 timeout 600 python tools/tc_trace.py C5 40 > gpurun_out/t2/trace_C5_$U0.txt 2>&1; done
for U0 in 0 200; do CR_TC_TRACE_U0=$U0 timeout 300 python tools/tc_trace.py C4 40 > gpurun_out/t2/trace_C4_$U0.txt 2>&1; done
CR_TC_TRACE_U0=0 timeout 300 python tools/tc_trace.py C3 40 > gpurun_out/t2/trace_C3_0.txt 2>&1
