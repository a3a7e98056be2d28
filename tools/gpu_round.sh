mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_tblock_gpu.py -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_tb.log 2>&1; echo pytest_exit=$?
grep -E "passed|failed|^E |FAILED" gpurun_out/pytest_tb.log | head -10
timeout 600 python tools/sweep.py --dtype f64 --depths 4 --tblocks 4,5 --tbdepths 4,6 > gpurun_out/sweep_tb64.log 2>&1; cat gpurun_out/sweep_tb64.log
timeout 600 python tools/sweep.py --dtype f32 --depths 4 --tblocks 5,6,8 --tbdepths 4 > gpurun_out/sweep_tb32.log 2>&1; cat gpurun_out/sweep_tb32.log
