# start-up rows (TSW_TB_STARTUP): TB / fused-energy / parity suites on the new default, interleaved A/B
# of su1 (skip the K(K+1) level-rows per item no output needs) vs su0, fused-energy cost, bench
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_tblock_gpu.py tests/test_energy_fused_gpu.py tests/test_peer_gpu.py -q -x -p no:cacheprovider > gpurun_out/pytest_tb.log 2>&1; echo pytest_tb=$?
tail -2 gpurun_out/pytest_tb.log
bash tools/ablibs.sh "su1 su0" "f64:10 f32:10 f64:8" 3 | tee gpurun_out/ab_startup.jsonl
for L in su1 su0; do
  out=$(TSW_LIB=abl/$L.so timeout 300 python tools/energy_fuse_time.py f64 10 2>&1 | tail -1)
  echo "{\"lib\": \"$L\", \"res\": $out}"
done | tee gpurun_out/ab_startup_energy.jsonl
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_su.json 2> gpurun_out/bench_su.err; echo bench=$?
