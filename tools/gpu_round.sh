mkdir -p gpurun_out
rm -f gpurun_out/pytest_imp.log gpurun_out/table1.log gpurun_out/launches_table1_scan.csv
timeout 1500 python -m pytest tests/test_implicit_gpu.py -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_imp.log 2>&1; echo pytest_exit=$?
grep -E "passed|failed|^E  |FAILED|Error" gpurun_out/pytest_imp.log | head -30
timeout 600 python tools/table1.py > gpurun_out/table1.log 2>&1; echo exit=$?
cut -c1-130 gpurun_out/table1.log
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_table1_scan.csv python tools/table1.py --sizes 4096 --dtypes f64,f32 --steps 3 --reps 1 > gpurun_out/ncu_t1.log 2>&1; echo ncu=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_imp_yc" --launch-skip 1 -c 1 -o gpurun_out/prof_impyc_f64 -f python tools/table1.py --sizes 4096 --dtypes f64 --steps 3 --reps 1 > gpurun_out/ncu_imp.log 2>&1; echo ncu2=$?
