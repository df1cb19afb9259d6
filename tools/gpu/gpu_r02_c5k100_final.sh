# round 2, session 4: C5 K=100 full-size parity record re-taken with the final kernels (column-sum chains,
# RED flushes, zero-tile GEMM2 skip); the fp64 oracle needs ~22 s per C5 iteration on the box's 16 cores
mkdir -p gpurun_out/c5k100
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c5k100/build.log 2>&1
timeout 3300 python tools/full_parity.py both C5 100 > gpurun_out/c5k100/full_parity_C5.log 2>&1
cp profiles/r02/parity_C5_K100.json gpurun_out/c5k100/ 2>/dev/null
