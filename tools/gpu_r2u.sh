mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_family_gpu.py -q -x -p no:cacheprovider > gpurun_out/pytest_fam.log 2>&1; echo "fam pytest=$? $(tail -1 gpurun_out/pytest_fam.log)"
timeout 300 python tools/diag_time.py f64 2>/dev/null | head -1
timeout 300 python tools/diag_time.py f32 2>/dev/null | head -1
