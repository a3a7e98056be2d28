# balanced partition of the temporally blocked pass: TB / fused-energy suites, interleaved A/B of
# TSW_OPT_TB_PARTITION 0 (round-robin items) vs 1 (auto: balanced on the bench), default bench
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_tblock_gpu.py tests/test_energy_fused_gpu.py -q -x -p no:cacheprovider > gpurun_out/pytest_tb.log 2>&1; echo pytest_tb=$?
tail -2 gpurun_out/pytest_tb.log
for r in 1 2 3; do for p in 0 1; do for c in f64:10 f32:10; do
  dt=${c%%:*}; K=${c#*:}
  out=$(TSW_AB_PART=$p timeout 300 python tools/abtest.py $dt $K 2 2>&1 | tail -1)
  echo "{\"round\": $r, \"part\": $p, \"case\": \"$c\", \"res\": $out}"
done; done; done | tee gpurun_out/ab_part.jsonl
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_part.json 2> gpurun_out/bench_part.err; echo bench=$?
# fused energy: one running sum per column (TSW_TB_EN_SPLIT=1, cur) vs one per thread (es0)
for r in 1 2; do for L in cur es0; do
  out=$(TSW_LIB=abl/$L.so timeout 300 python tools/energy_fuse_time.py f64 10 2>&1 | tail -1)
  echo "{\"round\": $r, \"lib\": \"$L\", \"res\": $out}"
done; done | tee gpurun_out/ab_ensplit.jsonl
