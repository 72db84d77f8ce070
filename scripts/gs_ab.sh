# A/B of two builds (vA, vB) and an env knob on vB: ENVK=SEGCONV_WIDE_BPROD VALS="0 1"
L=paper_2209_03704_b200
t() { timeout 120 python bench.py --config $1 --steps 20 --warmup 5 --no-baselines --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step']*1000,1))"; }
for r in 1 2; do
  cp $L/libsegconv_b200_vA.so $L/libsegconv_b200.so
  for c in ${CONFIGS:-C3 C5}; do echo "vA $c $(t $c)"; done
  cp $L/libsegconv_b200_vB.so $L/libsegconv_b200.so
  for g in ${VALS:-1}; do
    for c in ${CONFIGS:-C3 C5}; do echo "vB $ENVK=$g $c $(env ${ENVK:-X}=$g bash -c "$(declare -f t); t $c")"; done
  done
done
