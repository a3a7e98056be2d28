mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo smoke_exit=$?; tail -2 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$?
tail -4 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-also > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench_exit=$?
cat gpurun_out/bench_default.json; tail -3 gpurun_out/bench_default.err
