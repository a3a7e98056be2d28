# re-entry check: GPU suite, smoke, default bench; A/B of the fp64 K = 10 CTA shape (12 warps x 1 vs 6 warps x 2 per SM)
mkdir -p gpurun_out
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench=$?
bash tools/gpu_ab.sh "v0 w6" "f64:10" 2 2>&1 | tee gpurun_out/ab_w6.jsonl
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 1200 -p no:cacheprovider --durations=5 > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$?
tail -3 gpurun_out/pytest_gpu.log
