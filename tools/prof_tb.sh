mkdir -p gpurun_out
timeout 300 python tools/abtest.py f64 4 1 > gpurun_out/ab_plain.log 2>&1; echo plain=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_step2d_tb" --launch-skip 12 -c 1 -o gpurun_out/prof_tb4_f64 -f python tools/abtest.py f64 4 1 > gpurun_out/ncu_tb4.log 2>&1; echo ncu64=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_step2d_tb" --launch-skip 12 -c 1 -o gpurun_out/prof_tb8_f32 -f python tools/abtest.py f32 8 1 > gpurun_out/ncu_tb8.log 2>&1; echo ncu32=$?
