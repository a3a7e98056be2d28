# start-up rows fixed for the fp32 y-flux cache + output-row predicate / byte-stride pointer: full GPU
# suite, A/B vs the plain pass (su0), fused-energy cost, bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 1200 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu.log
bash tools/ablibs.sh "cur su0" "f64:10 f32:10 f64:8" 4 | tee gpurun_out/ab_startup3.jsonl
for L in cur su0; do
  out=$(TSW_LIB=abl/$L.so timeout 300 python tools/energy_fuse_time.py f64 10 2>&1 | tail -1)
  echo "{\"lib\": \"$L\", \"res\": $out}"
done | tee gpurun_out/ab_startup3_energy.jsonl
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_su3.json 2> gpurun_out/bench_su3.err; echo bench=$?
