for dbg in 0 1 8 9; do
 SEGCONV_TC_DEBUG=$dbg python scripts/layer_time.py 1024 11 128 3 3 0 ; SEGCONV_TC_DEBUG=$dbg NOFLUSH=1 python scripts/layer_time.py 1024 11 128 3 3 0
done
