# centre rows split into even / odd columns (TSW_TB_SPLIT_CEN = 1): TB / energy / peer suites on the
# split build, interleaved A/B against the default layout
mkdir -p gpurun_out
TSW_LIB=abl/split.so timeout 900 python -m pytest tests/test_tblock_gpu.py tests/test_energy_fused_gpu.py tests/test_peer_gpu.py -q -x -p no:cacheprovider > gpurun_out/ab_test_split.log 2>&1
echo "tests split rc=$? $(tail -1 gpurun_out/ab_test_split.log)"
bash tools/ablibs.sh "cur split" "f64:10 f32:10 f64:4" 3 | tee gpurun_out/ab_split_cen.jsonl
