# round-2 final evidence (start-up rows in the TB stencil): GPU suite, smoke, default bench, launch
# list, ncu --set full of the K = 10 passes (fp64, fp32, fp64 fused energy), workload lines
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 1200 -p no:cacheprovider --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$?
tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_bench.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/ncu_launches.log 2>&1; echo launches=$?
for dt in f64 f32; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_step2d_tb" --launch-skip 12 -c 1 \
    -o gpurun_out/prof_tb10_$dt -f python tools/abtest.py $dt 10 1 > gpurun_out/ncu_tb10_$dt.log 2>&1; echo ncu_$dt=$?
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_step2d_tb" -c 3 -o gpurun_out/prof_en10_f64 -f \
  python tools/en_one.py f64 10 > gpurun_out/ncu_en10.log 2>&1; echo ncu_en=$?
bash tools/gpu_workloads.sh
