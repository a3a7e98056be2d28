mkdir -p gpurun_out
timeout 300 python tools/debug_energy_fuse.py > gpurun_out/dbg_en.log 2>&1; echo dbg=$?
timeout 300 python tools/energy_fuse_time.py f64 8,4 > gpurun_out/en_f64.json 2>&1; echo t64=$?; tail -1 gpurun_out/en_f64.json
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_step2d_tb -c 3 -o gpurun_out/prof_en4 -f python tools/en_one.py f64 4 > gpurun_out/ncu_en4.log 2>&1; echo ncu=$?
