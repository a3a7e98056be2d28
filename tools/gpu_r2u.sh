mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_tblock_gpu.py tests/test_energy_fused_gpu.py tests/test_peer_gpu.py tests/test_peer_ipc_gpu.py tests/test_parity_gpu.py -q -x -p no:cacheprovider -k "not config3_full and not config5_batched" > gpurun_out/pytest_new.log 2>&1; echo "pytest=$? $(tail -1 gpurun_out/pytest_new.log)"
bash tools/abdepth.sh "cur new" "f64:8 f64:7 f64:6 f64:4 f32:8" 2 "0"
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_new.json 2> gpurun_out/bench_new.err; echo bench=$?
