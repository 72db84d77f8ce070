# A/B timing of two library builds on one config: libsegconv_b200_vA.so vs _vB.so
# usage: A=v25 B=v16 CONFIG=C3 bash scripts/ab_lib.sh
L=paper_2209_03704_b200
for i in 1 2 3; do
  for v in $A $B; do
    cp $L/libsegconv_b200_$v.so $L/libsegconv_b200.so
    echo -n "$v "; timeout 120 python bench.py --config ${CONFIG:-C3} --steps 20 --warmup 5 --no-baselines --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step']*1000)"
  done
done
