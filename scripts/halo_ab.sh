# pair kernel: im2col vs 2-D halo staging per GAN layer shape (batch 64, 4x4, p = 2)
for spec in "4 2048 1024" "8 1024 512" "16 512 256" "32 256 128" "64 128 64" "128 64 64" "32 128 64" "16 256 128" "64 64 64"; do
  set -- $spec
  a=$(timeout 120 python scripts/layer_time.py 64 $1 $2 $3 4 2 2>&1 | tail -1 | awk '{print $(NF-1)}')
  b=$(SEGCONV_WIDE_IM2COL=0 timeout 120 python scripts/layer_time.py 64 $1 $2 $3 4 2 2>&1 | tail -1 | awk '{print $(NF-1)}')
  echo "n=$1 $2->$3: im2col $a halo $b"
done
