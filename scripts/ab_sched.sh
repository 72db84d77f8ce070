# balanced unit schedule vs round-robin (SEGCONV_TC_DEBUG=64) on the C5 layers, C3, and the stack
for dbg in 0 64; do
  for L in "1024 4 1024 512 3 0" "1024 5 512 256 3 0" "1024 7 256 128 3 0" "128 16 512 256 4 0"; do
    SEGCONV_TC_DEBUG=$dbg python scripts/layer_time.py $L
  done
  SEGCONV_TC_DEBUG=$dbg python bench.py --steps 20 --warmup 5 --no-baselines --no-e2e > gpurun_out/st_$dbg.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/st_$dbg.json'));print('stack dbg=$dbg', d['ms_per_step'], [(l['layer'], l['ms']) for l in d['layers']], d['parity']['pass'])"
done
