mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/pytest_all.log 2>&1; echo pytest_exit=$?
tail -3 gpurun_out/pytest_all.log
grep -E "FAILED|Error" gpurun_out/pytest_all.log | head -10
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
