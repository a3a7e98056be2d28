mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_tblock_gpu.py tests/test_energy_fused_gpu.py tests/test_guards_gpu.py tests/test_peer_gpu.py -q -x -p no:cacheprovider > gpurun_out/pytest_ens.log 2>&1; echo "ens pytest=$? $(tail -1 gpurun_out/pytest_ens.log)"
timeout 300 python tools/energy_fuse_time.py f64 10,9,8 | tail -1
bash tools/ablibs.sh "cur ens" "f64:10" 2
for L in cur ens; do TSW_LIB=abl/$L.so timeout 300 python tools/energy_fuse_time.py f64 10 | tail -1; done
