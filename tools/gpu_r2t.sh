mkdir -p gpurun_out
TSW_LIB=abl/w12f.so timeout 900 python -m pytest tests/test_tblock_gpu.py tests/test_energy_fused_gpu.py -q -x -p no:cacheprovider > gpurun_out/pytest_w12f.log 2>&1; echo "w12f pytest=$? $(tail -1 gpurun_out/pytest_w12f.log)"
bash tools/abdepth.sh "cur w11 w12 w14 w12f" "f64:8 f32:8" 2 "4"
bash tools/abdepth.sh "w12" "f64:8" 1 "8"
