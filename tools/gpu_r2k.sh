mkdir -p gpurun_out
TSW_LIB=abl/p1.so timeout 1200 python -m pytest tests/test_tblock_gpu.py tests/test_energy_fused_gpu.py tests/test_peer_gpu.py -q -x -p no:cacheprovider > gpurun_out/pytest_p1.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_p1.log
bash tools/ablibs.sh "p0 p1" "f64:8 f32:8 f64:4" 3
