# round profiles: ncu launch lists (duration + DRAM bytes) per config, then one
# --set full capture of each hot kernel (each only after its plain run exits 0)
set -x
mkdir -p gpurun_out
for c in ${CONFIGS:-C2 C3 C4 C5}; do
python bench.py --config $c --steps 2 --warmup 3 --no-baselines --no-e2e > gpurun_out/plain_launch_$c.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$c.csv python bench.py --config $c --steps 2 --warmup 3 --no-baselines --no-e2e > gpurun_out/ncu_launch_$c.log 2>&1
echo launches $c=$?
done
for spec in ${FULL:-C2:fold_ts C3:wide_kernel}; do
  c=${spec%%:*}; k=${spec##*:}
  bash scripts/gpu_ncu.sh $c $k ${c,,}_${TAG:-r01}
done
