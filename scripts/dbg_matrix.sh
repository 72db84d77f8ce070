# diagnostics: C2 step time with parts of the fold kernel disabled (SEGCONV_TC_DEBUG bits)
for d in 0 1 2 4 8 6 14 15; do SEGCONV_TC_DEBUG=$d timeout 120 python bench.py --config ${CFG:-C2} --no-baselines --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"dbg $d\", round(d[\"ms_per_step\"]*1000,2), \"us\")"; done
