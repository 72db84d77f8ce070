# usage: bash scripts/gpu_ncu2.sh <tag> <kernel-regex> <launch-skip> -- <bench args...>
# plain run first (must exit 0), then one ncu --set full capture of one launch
mkdir -p gpurun_out
tag=$1; kre=$2; skip=$3; shift 4
python bench.py --steps 2 --warmup 3 --no-baselines --no-e2e --no-parity "$@" > gpurun_out/plain_$tag.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$kre -s $skip -c 1 -o /tmp/prof_$tag -f \
    python bench.py --steps 2 --warmup 3 --no-baselines --no-e2e --no-parity "$@" > gpurun_out/ncu_$tag.log 2>&1
echo ncu_$tag=$?
ncu -i /tmp/prof_$tag.ncu-rep --page raw --csv > gpurun_out/raw_$tag.csv 2>&1
ncu -i /tmp/prof_$tag.ncu-rep --page details --csv > gpurun_out/details_$tag.csv 2>&1
ncu -i /tmp/prof_$tag.ncu-rep --page source --csv > gpurun_out/source_$tag.csv 2>&1
sz=$(stat -c %s /tmp/prof_$tag.ncu-rep)
if [ "$sz" -lt 30000000 ]; then cp /tmp/prof_$tag.ncu-rep gpurun_out/; fi
