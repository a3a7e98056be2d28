mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_tblock_gpu.py tests/test_guards_gpu.py tests/test_peer_gpu.py -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_tb.log 2>&1; echo pytest_exit=$?
tail -2 gpurun_out/pytest_tb.log
timeout 600 python bench.py --workload config5 --steps 400 --no-cpu-baseline --no-e2e > gpurun_out/bench_config5.json 2> gpurun_out/bench_config5.err; echo c5=$?
timeout 600 python bench.py --workload config3 --steps 1000 --no-cpu-baseline --no-e2e > gpurun_out/bench_config3.json 2> gpurun_out/bench_config3.err; echo c3=$?
timeout 300 python tools/abtest.py f64 4 3 > gpurun_out/ab64.log 2>&1; cat gpurun_out/ab64.log
