# backward-pass benches (bench.py --pass backward) + a launch list of one
mkdir -p gpurun_out
for c in ${CONFIGS:-C3 C5a C5b C5c C2}; do
  timeout 600 python bench.py --config $c --pass backward --steps 10 --warmup 3 > gpurun_out/bench_bwd_$c.json 2> gpurun_out/bench_bwd_$c.err
  echo "bench bwd $c rc=$?"; tail -c 1500 gpurun_out/bench_bwd_$c.json | cut -c1-1500
done
if [ -n "$NCU" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    python bench.py --config C3 --pass backward --steps 2 --warmup 3 --no-baselines --no-e2e > gpurun_out/ncu_bwd_C3.csv 2>&1
  echo "ncu rc=$?"
fi
