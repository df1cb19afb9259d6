# round 2: same-box A/B -- GEMM1-only f16 (HEAD before the GEMM2 change, built into _ab/prev) vs GEMM1+GEMM2 f16
mkdir -p gpurun_out
python -c "import paper_1608_02227_b200.build as b; b.build()" > gpurun_out/build.log 2>&1
run() { d=$1; t=$2; shift 2; (cd $d && env "$@" timeout 600 python bench.py --config C5 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e) > gpurun_out/ab3_$t.json 2>&1; }
run _ab/prev prev1 X=0; run . new1 X=0; run _ab/prev prev2 X=0; run . new2 X=0
(cd _ab/prev && timeout 600 python bench.py --config C5 --steps 200 --warmup 5 --no-cpu-baseline --no-e2e) > gpurun_out/ab3_prev200.json 2>&1
timeout 600 python bench.py --config C5 --steps 200 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab3_new200.json 2>&1
