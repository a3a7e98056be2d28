mkdir -p gpurun_out
timeout 300 python tools/debug_energy_fuse.py > gpurun_out/dbg_en.log 2>&1; echo dbg=$?
timeout 300 ncu --section LaunchStats --section Occupancy --section SpeedOfLight --section WarpStateStats -k regex:k_step2d_tb -c 3 python tools/en_one.py f64 4 > gpurun_out/ncu_en4.txt 2>&1; echo ncu=$?
