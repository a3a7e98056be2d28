# round-2 final evidence, measurement half (the GPU suite and smoke ran green on this code in
# gpu_final4.sh): default bench, launch list, ncu --set full of the K = 10 passes exported to CSV
# (the reports themselves exceed gpurun's 64 MiB return), workload lines
mkdir -p gpurun_out
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_bench.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/ncu_launches.log 2>&1; echo launches=$?
prof() {  # name, command...
  local n=$1; shift
  timeout 600 ncu --set full --import-source on --clock-control none "$@" -o /tmp/$n -f > gpurun_out/$n.log 2>&1; echo $n=$?
  ncu -i /tmp/$n.ncu-rep --page raw --csv > gpurun_out/${n}_raw.csv 2>/dev/null
  ncu -i /tmp/$n.ncu-rep --page details --csv > gpurun_out/${n}_details.csv 2>/dev/null
}
prof ncu_tb10_f64 -k regex:"k_step2d_tb" --launch-skip 12 -c 1 python tools/abtest.py f64 10 1
prof ncu_tb10_f32 -k regex:"k_step2d_tb" --launch-skip 12 -c 1 python tools/abtest.py f32 10 1
prof ncu_en10_f64 -k regex:"k_step2d_tb" -c 3 python tools/en_one.py f64 10
bash tools/gpu_workloads.sh
du -sh gpurun_out
