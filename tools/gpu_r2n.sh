mkdir -p gpurun_out
TSW_LIB=abl/rowov.so timeout 1200 python -m pytest tests/test_tblock_gpu.py tests/test_peer_gpu.py tests/test_energy_fused_gpu.py -q -x -p no:cacheprovider > gpurun_out/pytest_rowov.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_rowov.log
bash tools/ablibs.sh "cur rowov" "f64:8 f32:8 f64:4 f32:4" 3
