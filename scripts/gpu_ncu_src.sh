# usage: bash scripts/gpu_ncu_src.sh <config> <kernel-regex> <tag>: ncu full + dense PC sampling
set -x
mkdir -p gpurun_out
cfg=$1; kre=$2; tag=$3; shift 3
python bench.py --config $cfg --steps 2 --warmup 3 --no-baselines "$@" > gpurun_out/plain_$tag.log 2>&1 && \
ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k regex:$kre -s 2 -c 1 -o /tmp/prof_$tag -f \
    python bench.py --config $cfg --steps 2 --warmup 3 --no-baselines "$@" > gpurun_out/ncu_$tag.log 2>&1
echo ncu=$?
ncu -i /tmp/prof_$tag.ncu-rep --page raw --csv > gpurun_out/raw_$tag.csv 2>&1
ncu -i /tmp/prof_$tag.ncu-rep --page source --csv > gpurun_out/source_$tag.csv 2>&1
ncu -i /tmp/prof_$tag.ncu-rep --page details --csv > gpurun_out/details_$tag.csv 2>&1
