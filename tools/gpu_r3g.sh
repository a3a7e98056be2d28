# fp64 y-flux cache for the first L levels only (TSW_TB_YCACHE_F64_LEVELS = 2, 4): TB / energy suites
# on each build, interleaved A/B against the default (no fp64 cache)
mkdir -p gpurun_out
for L in yc2 yc4; do
  TSW_LIB=abl/$L.so timeout 900 python -m pytest tests/test_tblock_gpu.py tests/test_energy_fused_gpu.py -q -x -p no:cacheprovider > gpurun_out/ab_test_$L.log 2>&1
  echo "tests $L rc=$? $(tail -1 gpurun_out/ab_test_$L.log)"
done
bash tools/ablibs.sh "cur yc2 yc4" "f64:10 f64:8" 3 | tee gpurun_out/ab_ycache_levels.jsonl
