mkdir -p gpurun_out
bash tools/abdepth.sh "mbyc mbycp" "f64:8 f64:4" 2 "4"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_step2d_tb" --launch-skip 12 -c 1 \
    -o gpurun_out/prof_mbyc -f env TSW_LIB=abl/mbyc.so python tools/abtest.py f64 8 1 > gpurun_out/ncu_mbyc.log 2>&1; echo ncu=$?
