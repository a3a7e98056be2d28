mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_energy_fused_gpu.py tests/test_tblock_gpu.py -q -x -p no:cacheprovider > gpurun_out/pytest_en.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_en.log
timeout 300 python tools/energy_fuse_time.py f64 8,4 > gpurun_out/en_f64.json 2>&1; echo t64=$?; cat gpurun_out/en_f64.json | tail -2
timeout 300 python tools/energy_fuse_time.py f32 8,4 > gpurun_out/en_f32.json 2>&1; echo t32=$?; cat gpurun_out/en_f32.json | tail -2
python -c "
import sys; sys.path.insert(0,'.')
from paper_2005_11931_b200 import tsw
for d,n in ((tsw.TSW_F64,'f64'),(tsw.TSW_F32,'f32')):
    print(n, tsw.tsw_alu_probe(0, d)/1e12, 'TOP/s')
"
