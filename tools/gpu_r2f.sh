mkdir -p gpurun_out
timeout 300 python tools/debug_energy_fuse.py > gpurun_out/dbg_en.log 2>&1; echo dbg=$?
timeout 300 python tools/energy_fuse_time.py f64 8,4 > gpurun_out/en_f64.json 2>&1; echo t64=$?; tail -1 gpurun_out/en_f64.json
timeout 300 python tools/energy_fuse_time.py f32 8,4 > gpurun_out/en_f32.json 2>&1; echo t32=$?; tail -1 gpurun_out/en_f32.json
timeout 900 python -m pytest tests/test_energy_fused_gpu.py -q -x -p no:cacheprovider > gpurun_out/pytest_en.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_en.log
