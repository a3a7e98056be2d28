# round-2 evidence: default bench line, launch list of the same command under ncu, --set full of the
# K = 8 passes (fp64, fp32) and of the fused-energy K = 4 pass, CPU oracle baseline plan
mkdir -p gpurun_out
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_bench.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/ncu_launches.log 2>&1; echo launches=$?
for dt in f64 f32; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_step2d_tb" --launch-skip 12 -c 1 \
    -o gpurun_out/prof_tb8_$dt -f python tools/abtest.py $dt 8 1 > gpurun_out/ncu_tb8_$dt.log 2>&1; echo ncu_$dt=$?
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_step2d_tb" -c 3 -o gpurun_out/prof_en4_f64 -f \
  python tools/en_one.py f64 4 > gpurun_out/ncu_en4.log 2>&1; echo ncu_en=$?
timeout 1200 python tools/cpu_baseline.py gpurun_out/cpu_baseline.jsonl > gpurun_out/cpu_baseline.log 2>&1; echo cpu=$?
