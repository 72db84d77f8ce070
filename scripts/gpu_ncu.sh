# usage: bash scripts/gpu_ncu.sh <config> <kernel-regex> <tag> [extra bench args]
set -x
mkdir -p gpurun_out
cfg=$1; kre=$2; tag=$3; shift 3
python bench.py --config $cfg --steps 2 --warmup 3 --no-baselines --no-e2e "$@" > gpurun_out/plain_$tag.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$kre -s 2 -c 1 -o /tmp/prof_$tag -f \
    python bench.py --config $cfg --steps 2 --warmup 3 --no-baselines --no-e2e "$@" > gpurun_out/ncu_$tag.log 2>&1
echo ncu=$?
ncu -i /tmp/prof_$tag.ncu-rep --page raw --csv > gpurun_out/raw_$tag.csv 2>&1
ncu -i /tmp/prof_$tag.ncu-rep --page details --csv > gpurun_out/details_$tag.csv 2>&1
ncu -i /tmp/prof_$tag.ncu-rep --page source --csv > gpurun_out/source_$tag.csv 2>&1
ls -la /tmp/prof_$tag.ncu-rep
sz=$(stat -c %s /tmp/prof_$tag.ncu-rep)
if [ "$sz" -lt 30000000 ]; then cp /tmp/prof_$tag.ncu-rep gpurun_out/; fi
