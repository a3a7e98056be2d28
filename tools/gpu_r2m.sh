mkdir -p gpurun_out
TSW_LIB=abl/pp.so timeout 1200 python -m pytest tests/test_tblock_gpu.py tests/test_energy_fused_gpu.py -q -x -p no:cacheprovider > gpurun_out/pytest_pp.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_pp.log
bash tools/ablibs.sh "p2 pp" "f64:8 f32:8 f64:4" 3
