# quick iteration: GPU tests, then benches of the given configs (default C2)
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
tail -5 gpurun_out/gpu_tests.log
for c in ${CONFIGS:-C2}; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-baselines > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo bench $c=$?; python -c "
import json; d=json.loads(open('gpurun_out/bench_$c.json').read().strip().splitlines()[-1]); print('$c', d['value'], 'us', d['ms_per_step']*1000, 'frac', d['roofline']['frac'], 'e2e', d['e2e']['value'], d['clocks'])"; done
