# eight vs four epilogue warps (SEGCONV_TC_DEBUG=256) on the forward pair kernel at one CTA per SM
for d in 0 256 0 256; do
  SEGCONV_TC_DEBUG=$d python bench.py --steps 30 --warmup 5 --no-baselines --no-e2e --no-parity > gpurun_out/st.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/st.json'));print('C5 dbg=$d', d['ms_per_step'], [(l['layer'], l['ms']) for l in d['layers']])"
  SEGCONV_TC_DEBUG=$d python bench.py --config C3 --steps 30 --warmup 5 --no-baselines --no-e2e --no-parity 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('C3 dbg=$d', d['ms_per_step'])"
done
for c in C5b C5c; do for d in 0 256; do
  SEGCONV_TC_DEBUG=$d python bench.py --config $c --pass backward --steps 10 --warmup 3 --no-baselines --no-e2e --no-parity 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$c bwd dbg=$d', d['ms_per_step'])"
done; done
