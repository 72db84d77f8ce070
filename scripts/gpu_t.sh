# usage: bash scripts/gpu_t.sh "<pytest args>" [bench configs...]
mkdir -p gpurun_out
timeout 1500 python -m pytest $1 > gpurun_out/t.log 2>&1; echo tests=$?
shift
for c in "$@"; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-baselines > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo bench $c=$?; done
