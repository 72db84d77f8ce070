# A/B timing of library builds: VARIANTS="vA vB" CONFIGS="C4 C5" EXTRA="--pass backward" bash scripts/ab4.sh
L=paper_2209_03704_b200
cp $L/libsegconv_b200.so /tmp/lib_current.so
for c in ${CONFIGS:-${CONFIG:-C3}}; do
for i in 1 2 3; do
  for v in $VARIANTS; do
    cp $L/libsegconv_b200_$v.so $L/libsegconv_b200.so
    echo -n "$c $v "; timeout 120 python bench.py --config $c $EXTRA --steps 20 --warmup 5 --no-baselines --no-e2e --no-parity 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step']*1000)"
  done
done
done
cp /tmp/lib_current.so $L/libsegconv_b200.so
