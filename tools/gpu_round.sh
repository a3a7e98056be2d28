mkdir -p gpurun_out
for w in config5 config3; do
timeout 900 python bench.py --workload $w --no-cpu-baseline --steps 500 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo "$w exit=$?"; cat gpurun_out/bench_$w.json | python -c "import json,sys; d=json.load(sys.stdin); print(d['config']['workload'], d['value'], d['roofline']['frac'], d.get('also',{}).get('value'), d.get('per_step_kernel',{}).get('value'), d['e2e']['value'])"; tail -2 gpurun_out/bench_$w.err
done
