mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$?
tail -4 gpurun_out/pytest_gpu.log
timeout 600 python tools/sweep.py --dtype f64 --depths 3,4,5 --rows 0,37,54,111,147 > gpurun_out/sweep_f64.log 2>&1
cat gpurun_out/sweep_f64.log
timeout 600 python tools/sweep.py --dtype f32 --depths 3,4,5 --rows 0,37,111 > gpurun_out/sweep_f32.log 2>&1
cat gpurun_out/sweep_f32.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench_exit=$?
cat gpurun_out/bench_default.json
