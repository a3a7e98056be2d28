# round 2, first call: box facts, the GPU suite, the default bench line, ncu of the TB passes
mkdir -p gpurun_out
(nproc; free -g; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv) > gpurun_out/box.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider --durations=25 > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench=$?
for dt in f64 f32; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_step2d_tb" --launch-skip 12 -c 1 \
    -o gpurun_out/prof_tb8_$dt -f python tools/abtest.py $dt 8 1 > gpurun_out/ncu_tb8_$dt.log 2>&1; echo ncu_$dt=$?
done
