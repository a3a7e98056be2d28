mkdir -p gpurun_out
timeout 900 python tools/debug_tb.py > gpurun_out/stress.log 2>&1; cat gpurun_out/stress.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$?
grep -E "passed|failed|^E |FAILED" gpurun_out/pytest_gpu.log | head -10
for k in 1 2 3; do timeout 600 python -m pytest tests/test_tblock_gpu.py::test_tblock_bench_shape_sampled -q -p no:cacheprovider 2>&1 | tail -1; done
