# Round-2 measurement set: every config's bench line, the reference arm, the
# C5 launch list and one full capture of the C5 dominant kernel (layer a).
mkdir -p gpurun_out/r02
for c in C5 C2 C1 C3 C4 C3f32; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/r02/bench_$c.json 2> gpurun_out/r02/bench_$c.err; echo bench $c=$?
done
for c in C5 C2 C4; do
  timeout 600 python bench.py --impl reference --config $c --steps 3 --warmup 1 > gpurun_out/r02/ref_$c.json 2> gpurun_out/r02/ref_$c.err; echo ref $c=$?
done
for c in C3 C5a C5b C5c C2 C4; do
  timeout 600 python bench.py --config $c --pass backward --steps 10 --warmup 3 > gpurun_out/r02/bwd_$c.json 2> gpurun_out/r02/bwd_$c.err; echo bwd $c=$?
done
for c in C5 C2 C4 C3 C1; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/r02/launches_$c.csv python bench.py --config $c --steps 2 --warmup 3 --no-baselines --no-e2e --no-parity > /dev/null 2>&1; echo launches $c=$?
done
# full captures of the pair kernel (layers a and c of the C5 stack) after the
# im2col pipeline changes
bash scripts/gpu_ncu2.sh c5a_r02b wide_kernel 3 -- --config C5a; mv gpurun_out/*_c5a_r02b.* gpurun_out/r02/ 2>/dev/null
bash scripts/gpu_ncu2.sh c5c_r02b wide_kernel 3 -- --config C5c; mv gpurun_out/*_c5c_r02b.* gpurun_out/r02/ 2>/dev/null
