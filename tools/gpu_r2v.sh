mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_tblock_gpu.py tests/test_energy_fused_gpu.py tests/test_peer_gpu.py -q -x -p no:cacheprovider > gpurun_out/pytest_k10.log 2>&1; echo "pytest=$? $(tail -1 gpurun_out/pytest_k10.log)"
bash tools/abdepth.sh "k10" "f64:8 f64:9 f64:10 f32:8 f32:9 f32:10" 2 "0"
