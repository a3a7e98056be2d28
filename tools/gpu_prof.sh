mkdir -p gpurun_out
timeout 120 python tools/table1.py --sizes 4096 --dtypes f64 --steps 3 --reps 1 > gpurun_out/t1_plain.log 2>&1 && \
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"^k_imp_(yc|x)$" --launch-skip 2 -c 2 -o gpurun_out/prof_imp_final_f64 -f python tools/table1.py --sizes 4096 --dtypes f64 --steps 3 --reps 1 > gpurun_out/ncu_imp.log 2>&1; echo ncu=$?
