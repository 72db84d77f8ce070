set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tc.py -q -x > gpurun_out/tc_tests.log 2>&1; echo tc=$?
for c in ${CONFIGS:-C3 C5}; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-baselines > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo bench $c=$?; done
SEGCONV_TC_TRACE=1 python scripts/trace_tc.py C3 > gpurun_out/trace_c3.txt 2>&1
