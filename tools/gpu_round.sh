mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_tblock_gpu.py tests/test_parity_gpu.py -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_tb.log 2>&1; echo pytest_exit=$?
tail -2 gpurun_out/pytest_tb.log
timeout 300 python tools/sweep.py --dtype f64 --steps 200 --depths 4 --tblocks 4,5,6 --tbdepths 4 > gpurun_out/sweep64.log 2>&1; echo s64=$?
timeout 300 python tools/sweep.py --dtype f32 --steps 200 --depths 4 --tblocks 5,6,8 --tbdepths 4 > gpurun_out/sweep32.log 2>&1; echo s32=$?
grep '"tb"' gpurun_out/sweep64.log gpurun_out/sweep32.log | cut -c1-200
