mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_tblock_gpu.py tests/test_energy_fused_gpu.py tests/test_peer_gpu.py tests/test_parity_gpu.py -q -x -p no:cacheprovider -k "f32 or tblock or fused or peer or loopback" > gpurun_out/pytest_sp.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_sp.log
bash tools/ablibs.sh "ns sp" "f32:8 f32:6 f32:4" 2
