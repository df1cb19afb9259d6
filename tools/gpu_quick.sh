mkdir -p gpurun_out
b() { tag=$1; shift; env "$@" timeout 300 python bench.py --no-cpu-baseline --no-e2e $CFG > gpurun_out/q_$tag.json 2> gpurun_out/q_$tag.err; }
CFG="--config C4"; b C4 X=1; b C4b X=1
CFG="--config C5 --steps 60"; b C5 X=1
CFG="--config C3"; b C3 X=1
