mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_implicit_gpu.py -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_imp.log 2>&1; echo pytest_exit=$?
grep -E "passed|failed|^E  |FAILED" gpurun_out/pytest_imp.log | head -20
