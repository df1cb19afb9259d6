# round 2: C3 pass investigation -- ring depths, L2 policy, ncu of one launch
mkdir -p gpurun_out
python -c "import paper_1608_02227_b200.build as b; b.build()" > gpurun_out/build.log 2>&1
run() { echo -n "$* : "; env "$@" timeout 300 python bench.py --config C3 --no-cpu-baseline --no-e2e --steps 2000 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,2), 'us', round(d['roofline']['frac'],4), round(d['roofline']['avg_launch_ms']*1e3,2), 'us')"; }
{
run X=0
run CR_TC_STAGES=6 CR_TC_G1STAGES=2 CR_TC_G2STAGES=2
run CR_TC_STAGES=4
run CR_TC_THETA_L2=3
run CR_TC_THETA_L2=1
run CR_TC_THETA_L2=2
run CR_TC_POLL_NS=0
run CR_TC_G1_F16=1
} > gpurun_out/c3_sweep.txt 2>&1
A="--config C3 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline"
timeout 600 python bench.py $A > gpurun_out/c3_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pass_tc -s 10 -c 1 -o gpurun_out/prof_C3 python bench.py $A > gpurun_out/ncu_c3.log 2>&1
