for hc in 0.65 0.8 0.9 1.0; do
  for rep in 1 2; do
  XSCHED_HALF=$hc python bench.py --steps 30 --warmup 5 --no-baselines --no-e2e --no-parity > gpurun_out/st.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/st.json'));print('stack hc=$hc', d['ms_per_step'], [(l['layer'], l['ms']) for l in d['layers']])"
  done
done
SEGCONV_TC_DEBUG=64 python bench.py --steps 30 --warmup 5 --no-baselines --no-e2e --no-parity > gpurun_out/st.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/st.json'));print('stack RR', d['ms_per_step'], [(l['layer'], l['ms']) for l in d['layers']])"
for hc in 0.65 1.0; do XSCHED_HALF=$hc python bench.py --config C3 --steps 30 --warmup 5 --no-baselines --no-e2e --no-parity > gpurun_out/st.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/st.json'));print('C3 hc=$hc', d['ms_per_step'])"; done
SEGCONV_TC_DEBUG=64 python bench.py --config C3 --steps 30 --warmup 5 --no-baselines --no-e2e --no-parity > gpurun_out/st.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/st.json'));print('C3 RR', d['ms_per_step'])"
