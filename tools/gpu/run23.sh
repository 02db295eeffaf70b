timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c3.json 2>gpurun_out/bench_c3.err; cat gpurun_out/bench_c3.json; tail -2 gpurun_out/bench_c3.err
for S in 1024 2048 4096 8192 16384 32768; do
  timeout 600 python bench.py --config c5 --seq $S --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5 S=%d'%d['config']['S'], round(d['value'],1), 'TF/s', round(d['ms_per_step'],3),'ms', 'e2e', round(d['e2e']['value'],1), 'trip', d['schedule_realized']['measured_clk_per_trip'])"
done
