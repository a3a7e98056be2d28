mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_family_l2 -c 1 -f -o gpurun_out/prof_fam_f64 python tools/fam_one.py f64 > gpurun_out/ncu_fam.log 2>&1; echo "ncu rc=$?"
