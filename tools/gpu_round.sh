mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_tblock_gpu.py tests/test_family_gpu.py tests/test_guards_gpu.py -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_e.log 2>&1; echo pytest_exit=$?
tail -2 gpurun_out/pytest_e.log
timeout 300 python bench.py --steps 200 --warmup 3 --no-cpu-baseline --no-also --no-e2e > gpurun_out/b_short.json 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"k_energy2d" --csv --log-file gpurun_out/launches_energy.csv python bench.py --steps 200 --warmup 3 --no-cpu-baseline --no-also --no-e2e > gpurun_out/ncu_e.log 2>&1; echo ncu=$?
