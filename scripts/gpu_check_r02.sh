mkdir -p gpurun_out/s3
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s3/gputest.log 2>&1; echo gputest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s3/smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py > gpurun_out/s3/bench_default.json 2> gpurun_out/s3/bench_default.err; echo bench=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/s3/ref.json 2> gpurun_out/s3/ref.err; echo ref=$?
tail -3 gpurun_out/s3/gputest.log; cat gpurun_out/s3/bench_default.json | head -c 1500
