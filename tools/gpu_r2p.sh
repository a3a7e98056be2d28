mkdir -p gpurun_out
TSW_LIB=abl/mbyc.so timeout 1200 python -m pytest tests/test_tblock_gpu.py tests/test_energy_fused_gpu.py -q -x -p no:cacheprovider -k "not f32" > gpurun_out/pytest_mbyc.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_mbyc.log
bash tools/abdepth.sh "cur minb1 mbyc" "f64:8 f64:4" 2 "4 8"
