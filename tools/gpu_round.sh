mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_implicit_gpu.py -q -x --timeout 120 -p no:cacheprovider > gpurun_out/pytest_imp.log 2>&1; echo pytest_exit=$?
tail -2 gpurun_out/pytest_imp.log; grep -E "^E  " gpurun_out/pytest_imp.log | head -5
for xr in 1 2 1 2; do timeout 120 python tools/table1.py --sizes 4096 --xrows $xr 2>&1 | cut -c1-140; done
