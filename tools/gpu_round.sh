mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench_exit=$?
cat gpurun_out/bench_default.json; tail -3 gpurun_out/bench_default.err
timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-also > gpurun_out/plain.log 2>&1 && \
timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-also --dtype f32 > gpurun_out/plain32.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_f64.csv python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-also > gpurun_out/ncu_launches.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step2d_tma -s 60 -c 1 -o gpurun_out/prof_tma_f64 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-also > gpurun_out/ncu_full.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step2d_tma -s 60 -c 1 -o gpurun_out/prof_tma_f32 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-also --dtype f32 > gpurun_out/ncu_full32.log 2>&1; echo ncu_exit=$?
ls gpurun_out
