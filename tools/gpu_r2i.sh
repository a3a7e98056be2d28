mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_peer_gpu.py tests/test_peer_ipc_gpu.py tests/test_energy_fused_gpu.py tests/test_tblock_gpu.py -q -x -p no:cacheprovider > gpurun_out/pytest_i.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_i.log
timeout 300 python tools/energy_fuse_time.py f64 8,4 > gpurun_out/en_f64.json 2>&1; tail -1 gpurun_out/en_f64.json
