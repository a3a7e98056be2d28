# bench lines of the other workloads (profiles/r02): config 5 ε family, config 3, the full 32768² grid
# (strong-scaling input), the paper's implicit Table-1 set-up, and a sustained 2000-step line
mkdir -p gpurun_out
for wl in config5 config3; do
  for dt in f64 f32; do
    timeout 900 python bench.py --workload $wl --dtype $dt --steps 200 --warmup 5 --no-cpu-baseline --no-also > gpurun_out/bench_${wl}_$dt.json 2> gpurun_out/bench_${wl}_$dt.err; echo $wl $dt=$?
  done
done
timeout 900 python bench.py --scaling strong --steps 100 --warmup 5 --no-cpu-baseline --no-also > gpurun_out/bench_strong.json 2> gpurun_out/bench_strong.err; echo strong=$?
for dt in f64 f32; do
  timeout 900 python bench.py --workload table1 --dtype $dt --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_table1_$dt.json 2> gpurun_out/bench_table1_$dt.err; echo table1 $dt=$?
done
timeout 900 python bench.py --steps 2000 --warmup 5 --no-cpu-baseline --no-also --no-e2e > gpurun_out/bench_sustained_2000.json 2> gpurun_out/bench_sustained.err; echo sustained=$?
