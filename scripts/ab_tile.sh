# tc-tile: three CTAs per SM (default when the shared memory allows) vs two (SEGCONV_TC_DEBUG=128)
for d in 0 128; do
  SEGCONV_TC_DEBUG=$d SEGCONV_TC_TRACE=1 NOFLUSH=1 python scripts/trace_tile.py 2>&1 | sed -n 2,4p
  for r in 1 2; do
  SEGCONV_TC_DEBUG=$d python bench.py --steps 30 --warmup 5 --no-baselines --no-e2e --no-parity > gpurun_out/st.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/st.json'));print('stack dbg=$d', d['ms_per_step'], [(l['layer'], l['ms']) for l in d['layers']])"
  done
done
