bash scripts/gpu_ncu2.sh c5c wide_kernel 3 -- --config C5c
bash scripts/gpu_ncu2.sh c5d tile_kernel 3 -- --config C5d
bash scripts/gpu_ncu2.sh c5c128 wide_kernel 3 -- --config C5c --batch 128
