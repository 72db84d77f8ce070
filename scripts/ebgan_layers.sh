# per-layer times of the EB-GAN preset (batch 64, 4x4, p = 2, bf16)
for spec in "4 2048 1024" "8 1024 512" "16 512 256" "32 256 128" "64 128 64" "128 64 64"; do
  set -- $spec
  echo -n "n=$1 $2->$3: "; timeout 120 python scripts/layer_time.py 64 $1 $2 $3 4 2 2>&1 | tail -1
done
