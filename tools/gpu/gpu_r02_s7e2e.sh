# round 2, session 7: run-to-run spread of the C4 e2e line at the driver's K = 20 (three runs)
mkdir -p gpurun_out/s7e2e
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s7e2e/build.log 2>&1
for i in 1 2 3; do
  timeout 300 python bench.py --config C4 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/s7e2e/C4_$i.json 2> gpurun_out/s7e2e/C4_$i.err
done
