mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_guards_gpu.py -q --timeout 120 -p no:cacheprovider > gpurun_out/pytest_guard.log 2>&1; echo pytest_exit=$?
tail -15 gpurun_out/pytest_guard.log
