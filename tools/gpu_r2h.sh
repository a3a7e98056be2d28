mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_guards_gpu.py tests/test_family_gpu.py tests/test_energy_fused_gpu.py tests/test_peer_ipc_gpu.py -q -x -p no:cacheprovider > gpurun_out/pytest_h.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_h.log
TSW_LIB=abl/v5.so timeout 600 python -m pytest tests/test_tblock_gpu.py -q -x -p no:cacheprovider > gpurun_out/ab_test_v5.log 2>&1; echo "v5 tests $? $(tail -1 gpurun_out/ab_test_v5.log)"
bash tools/ablibs.sh "v0 v5" "f64:6 f64:8" 3
