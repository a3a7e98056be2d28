mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$?
grep -E "passed|failed|^E |FAILED" gpurun_out/pytest_gpu.log | head -30
