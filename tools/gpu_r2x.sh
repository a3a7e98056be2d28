mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_energy2d|k_wave2" -c 2 -f -o gpurun_out/prof_diag_f32 python tools/diag_one.py f32 > gpurun_out/ncu_diag.log 2>&1; echo "ncu rc=$?"
