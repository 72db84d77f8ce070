# A/B/C/D timing of library builds: VARIANTS="vA vB" CONFIG=C4 bash scripts/ab4.sh
L=paper_2209_03704_b200
cp $L/libsegconv_b200.so /tmp/lib_current.so
for i in 1 2 3; do
  for v in $VARIANTS; do
    cp $L/libsegconv_b200_$v.so $L/libsegconv_b200.so
    echo -n "$v "; timeout 120 python bench.py --config ${CONFIG:-C3} --steps 20 --warmup 5 --no-baselines --no-e2e --no-parity 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step']*1000)"
  done
done
cp /tmp/lib_current.so $L/libsegconv_b200.so
