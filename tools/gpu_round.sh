mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_tblock_gpu.py tests/test_parity_gpu.py -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_tb.log 2>&1; echo pytest_exit=$?
tail -2 gpurun_out/pytest_tb.log
timeout 600 python bench.py --workload config5 --steps 400 --no-cpu-baseline --no-e2e > gpurun_out/bench_config5.json 2> gpurun_out/bench_config5.err; echo c5=$?
timeout 600 python bench.py --workload config3 --steps 1000 --no-cpu-baseline --no-e2e > gpurun_out/bench_config3.json 2> gpurun_out/bench_config3.err; echo c3=$?
