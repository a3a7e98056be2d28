mkdir -p gpurun_out
timeout 300 python bench.py --workload table1 --steps 100 --warmup 5 > gpurun_out/bench_table1_f64.json 2> gpurun_out/bench_table1_f64.err; echo f64=$?
timeout 300 python bench.py --workload table1 --steps 100 --warmup 5 --dtype f32 --no-cpu-baseline > gpurun_out/bench_table1_f32.json 2> gpurun_out/bench_table1_f32.err; echo f32=$?
tail -3 gpurun_out/bench_table1_f64.err
