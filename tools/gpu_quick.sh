mkdir -p gpurun_out
b() { tag=$1; shift; env "$@" timeout 300 python bench.py --no-cpu-baseline --no-e2e $CFG > gpurun_out/q_$tag.json 2> gpurun_out/q_$tag.err; }
CFG="--config C4"; b C4_p0 CR_TC_POLL_NS=0; b C4_p32 CR_TC_POLL_NS=32; b C4_p64 CR_TC_POLL_NS=64; b C4_p200 CR_TC_POLL_NS=200; b C4_p1000 CR_TC_POLL_NS=1000
CFG="--config C5 --steps 60"; b C5_p0 CR_TC_POLL_NS=0; b C5_p64 CR_TC_POLL_NS=64; b C5_p200 CR_TC_POLL_NS=200
CFG="--config C3"; b C3_p0 CR_TC_POLL_NS=0; b C3_p64 CR_TC_POLL_NS=64
