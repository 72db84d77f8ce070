# round-end refresh of the secondary bench lines (backward, GAN presets, C3 fp32)
mkdir -p gpurun_out
: > gpurun_out/bench_backward.jsonl; : > gpurun_out/bench_gan.jsonl; : > gpurun_out/bench_c3f32.jsonl
for c in C2 C3 C5a C5b C5c C4; do
  timeout 300 python bench.py --config $c --pass backward --steps 20 --warmup 5 2>gpurun_out/bwd_$c.err | tail -1 >> gpurun_out/bench_backward.jsonl
done
for g in dcgan artgan gpgan ebgan; do
  timeout 300 python bench.py --config gan:$g --steps 20 --warmup 5 2>gpurun_out/gan_$g.err | tail -1 >> gpurun_out/bench_gan.jsonl
done
timeout 300 python bench.py --config C3f32 --steps 20 --warmup 5 2>gpurun_out/c3f32.err | tail -1 >> gpurun_out/bench_c3f32.jsonl
