# diagnostics: wide-kernel step time with parts disabled (SEGCONV_TC_DEBUG bits:
# 8 no MMA, 16 no weight TMA, 32 no halo TMA, 1 no stores)
for d in 0 8 16 32 48 56 1; do SEGCONV_TC_DEBUG=$d timeout 120 python bench.py --config ${CFG:-C3} --no-baselines --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"dbg $d\", round(d[\"ms_per_step\"]*1000,2), \"us\")"; done
