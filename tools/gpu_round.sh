mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_implicit_gpu.py tests/test_guards_gpu.py -q -x --timeout 120 -p no:cacheprovider > gpurun_out/pytest_imp.log 2>&1; echo pytest_exit=$?
tail -2 gpurun_out/pytest_imp.log; grep -E "^E  " gpurun_out/pytest_imp.log | head -5
timeout 300 python bench.py --workload table1 --steps 100 > gpurun_out/bench_table1_f64.json 2> gpurun_out/bench_table1.err; echo t1=$?
timeout 300 python bench.py --workload table1 --steps 100 --dtype f32 --no-cpu-baseline > gpurun_out/bench_table1_f32.json 2>> gpurun_out/bench_table1.err; echo t1f32=$?
