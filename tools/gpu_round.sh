mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$?
tail -30 gpurun_out/pytest_gpu.log | grep -E "passed|failed|Error|assert|FAILED" | head -30
