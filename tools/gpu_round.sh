mkdir -p gpurun_out
rm -f gpurun_out/pytest_imp.log gpurun_out/table1.log gpurun_out/launches_table1_scan.csv
timeout 240 python -m pytest tests/test_implicit_gpu.py -q -x --timeout 60 -p no:cacheprovider > gpurun_out/pytest_imp.log 2>&1; echo pytest_exit=$?
grep -E "passed|failed|^E  |FAILED|Error|Timeout" gpurun_out/pytest_imp.log | head -30
timeout 120 python tools/table1.py > gpurun_out/table1.log 2>&1; echo exit=$?
cut -c1-130 gpurun_out/table1.log
timeout 120 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_table1_scan.csv python tools/table1.py --sizes 4096 --dtypes f64,f32 --steps 3 --reps 1 > gpurun_out/ncu_t1.log 2>&1; echo ncu=$?
