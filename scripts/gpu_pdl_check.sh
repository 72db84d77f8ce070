# fold-ts / ring kernels launched with programmatic stream serialization:
# their parity tests and the C2 / C4 bench lines
mkdir -p gpurun_out/pdl
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_range.py tests/test_gpu_guardbands.py tests/test_gpu_parity.py -x -q > gpurun_out/pdl/tests.log 2>&1; echo tests=$?
for c in C2 C4 C2 C4; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-baselines >> gpurun_out/pdl/bench_$c.json 2> gpurun_out/pdl/bench_$c.err; echo bench $c=$?
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/pdl/launches_C2.csv python bench.py --config C2 --steps 2 --warmup 3 --no-baselines --no-e2e --no-parity > /dev/null 2>&1; echo launches=$?
tail -2 gpurun_out/pdl/tests.log
