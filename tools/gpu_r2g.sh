mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_energy_fused_gpu.py tests/test_tblock_gpu.py tests/test_peer_gpu.py tests/test_peer_ipc_gpu.py tests/test_parity_gpu.py -q -x -p no:cacheprovider -k "not config3_full and not config4_full and not config5_batched" > gpurun_out/pytest_slab.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_slab.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench=$?
