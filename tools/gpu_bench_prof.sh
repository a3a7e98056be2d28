# Round bench line + the ncu evidence behind it (one GPU): the default bench, one `--set full`
# capture per precision of a steady-state temporally blocked pass on the bench workload, and the
# launch list of a short bench run.  Outputs under gpurun_out/.
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench=$?
for dt in f64 f32; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_step2d_tb" --launch-skip 12 -c 1 \
    -o gpurun_out/prof_tb8_$dt -f python tools/abtest.py $dt 8 1 > gpurun_out/ncu_tb8_$dt.log 2>&1; echo ncu_$dt=$?
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_bench.csv python bench.py --steps 200 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/ncu_launches.log 2>&1; echo launches=$?
