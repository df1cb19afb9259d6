# round 2: C5 K=200 full-size parity record (fp64 oracle on the box's host cores, 64 GiB in place, ~90 min),
# then the launch lists of the default bench command with room for the pass launches
mkdir -p gpurun_out
python -c "import paper_1608_02227_b200.build as b; b.build()" > gpurun_out/build.log 2>&1
timeout 7000 python tools/full_parity.py both C5 200 > gpurun_out/full_parity_C5.log 2>&1
for C in C5 C4; do
  A="--config $C --steps 20 --warmup 5 --no-e2e --no-cpu-baseline"
  timeout 600 python bench.py $A > gpurun_out/plain3_$C.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches3_$C.csv python bench.py $A > gpurun_out/ncu3_$C.log 2>&1
done
