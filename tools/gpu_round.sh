mkdir -p gpurun_out
timeout 600 python tools/sweep.py --dtype f64 --depths 4,6,8,12,16 --rows 0,128 --reg > gpurun_out/sweep_f64.log 2>&1; echo sweep_exit=$?
cat gpurun_out/sweep_f64.log
timeout 600 python tools/sweep.py --dtype f32 --depths 4,6,8,12 --rows 0 > gpurun_out/sweep_f32.log 2>&1
cat gpurun_out/sweep_f32.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$?
tail -8 gpurun_out/pytest_gpu.log
