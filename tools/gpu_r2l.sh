mkdir -p gpurun_out
TSW_LIB=abl/p2.so timeout 1200 python -m pytest tests/test_tblock_gpu.py tests/test_peer_gpu.py -q -x -p no:cacheprovider > gpurun_out/pytest_p2.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_p2.log
bash tools/ablibs.sh "p1 p2" "f64:8 f32:8 f64:4" 3
