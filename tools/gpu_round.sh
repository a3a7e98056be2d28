mkdir -p gpurun_out
timeout 600 python tools/sweep.py --dtype f64 --depths 4 --tblocks 4,5,6 --tbdepths 4 > gpurun_out/sweep_tb64.log 2>&1; cat gpurun_out/sweep_tb64.log
timeout 600 python tools/sweep.py --dtype f32 --depths 4 --tblocks 4,5,6 --tbdepths 4 > gpurun_out/sweep_tb32.log 2>&1; cat gpurun_out/sweep_tb32.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$?
grep -E "passed|failed|^E |FAILED" gpurun_out/pytest_gpu.log | head -20
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench_exit=$?
cat gpurun_out/bench_default.json; tail -3 gpurun_out/bench_default.err
