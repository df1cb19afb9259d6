# round 2: fused reduce+prologue rows per block (auto: 8 for small N, 32 for large) + the full GPU suite
mkdir -p gpurun_out
python -c "import paper_1608_02227_b200.build as b; b.build()" > gpurun_out/build.log 2>&1
run() { t=$1; C=$2; S=$3; shift 3; env "$@" timeout 600 python bench.py --config $C --steps $S --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r_${t}_${C}.json 2>&1; }
run auto C3 2000 X=0; run rpb32 C3 2000 CR_FUSE_RPB=32; run nofuse C3 2000 CR_NO_FUSE=1
run auto C4 20 X=0; run rpb32 C4 20 CR_FUSE_RPB=32
run auto C5 20 X=0; run rpb8 C5 20 CR_FUSE_RPB=8
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
