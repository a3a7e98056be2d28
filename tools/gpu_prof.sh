mkdir -p gpurun_out
timeout 200 python tools/sweep.py --dtype f32 --steps 20 --depths 4 --tblocks 8 --tbdepths 4 > gpurun_out/sweep_plain.log 2>&1; echo plain=$?
timeout 400 ncu --set full --import-source on --clock-control none -k regex:"k_step2d_tb" --launch-skip 3 -c 1 -o gpurun_out/prof_tb8_f32 -f python tools/sweep.py --dtype f32 --steps 20 --depths 4 --tblocks 8 --tbdepths 4 > gpurun_out/ncu_tb.log 2>&1; echo ncu=$?
