mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_energy_fused_gpu.py tests/test_parity_gpu.py -q -x -p no:cacheprovider > gpurun_out/pytest_en2d.log 2>&1; echo "en2d pytest=$? $(tail -1 gpurun_out/pytest_en2d.log)"
for L in cur en3s; do echo $L; TSW_LIB=abl/$L.so timeout 300 python tools/diag_time.py f64 2>/dev/null | cut -c1-200; TSW_LIB=abl/$L.so timeout 300 python tools/diag_time.py f32 2>/dev/null | cut -c1-200; done
echo new; timeout 300 python tools/diag_time.py f64 2>/dev/null | cut -c1-200; timeout 300 python tools/diag_time.py f32 2>/dev/null | cut -c1-200
