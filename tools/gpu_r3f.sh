# fp32 passes of 11 / 12 levels: TB / energy / slab suites, interleaved per-pass timing of K = 10, 11, 12
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_tblock_gpu.py tests/test_energy_fused_gpu.py tests/test_peer_gpu.py tests/test_parity_gpu.py -q -x -p no:cacheprovider > gpurun_out/pytest_k12.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_k12.log
for r in 1 2 3; do timeout 300 python tools/abtest.py f32 10,11,12 2 | tail -1; done | tee gpurun_out/ab_f32_depth.jsonl
