# The torchrun / NCCL path of bench.py on real hardware at world size 1 (the
# pool has one GPU per box): the driver's SCALE launch form, both arms, and
# the data-parallel backward step
mkdir -p gpurun_out/dist
export NCCL_DEBUG=INFO
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29531 \
  bench.py --gpus 1 --dist --steps 10 --warmup 3 > gpurun_out/dist/fwd.json 2> gpurun_out/dist/fwd.err; echo fwd=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29532 \
  bench.py --impl reference --gpus 1 --steps 2 --warmup 1 > gpurun_out/dist/ref.json 2> gpurun_out/dist/ref.err; echo ref=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 1 --dist --config C5a --pass backward --steps 5 --warmup 3 > gpurun_out/dist/bwd.json 2> gpurun_out/dist/bwd.err; echo bwd=$?
grep -m3 "NCCL INFO" gpurun_out/dist/fwd.err; true
