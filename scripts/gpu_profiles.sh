set -x
mkdir -p gpurun_out
for c in C2 C3 C4; do
python bench.py --config $c --steps 2 --warmup 3 --no-baselines > gpurun_out/plain_launch_$c.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$c.csv python bench.py --config $c --steps 2 --warmup 3 --no-baselines > gpurun_out/ncu_launch_$c.log 2>&1
echo launches $c=$?
done
bash scripts/gpu_ncu.sh C2 tc_fold c2_r01
bash scripts/gpu_ncu.sh C3 tc_halo c3_r01
