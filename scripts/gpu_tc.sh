set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tc.py -q -x > gpurun_out/tc_tests.log 2>&1; echo tc=$?
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/parity_tests.log 2>&1; echo parity=$?
for c in C2 C3 C5 C4; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-baselines > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo bench $c=$?; done
bash scripts/gpu_ncu.sh C2 tc_halo c2_tc2
bash scripts/gpu_ncu.sh C3 tc_halo c3_tc2
