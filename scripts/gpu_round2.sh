set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err; echo bench=$?
timeout 300 python bench.py --config C2 --steps 20 --warmup 5 > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err; echo benchC2=$?
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_C5.json 2>&1; echo ref=$?
