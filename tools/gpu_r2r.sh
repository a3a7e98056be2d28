mkdir -p gpurun_out
for L in w10yc w12; do TSW_LIB=abl/$L.so timeout 900 python -m pytest tests/test_tblock_gpu.py -q -x -p no:cacheprovider -k "not f32" > gpurun_out/pytest_$L.log 2>&1; echo "$L pytest=$? $(tail -1 gpurun_out/pytest_$L.log)"; done
bash tools/abdepth.sh "cur mbyc w10yc w12" "f64:8 f64:4" 2 "4"
