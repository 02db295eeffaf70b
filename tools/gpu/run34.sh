timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c3.json 2>gpurun_out/bench_c3.err; python -c "import json; d=json.load(open('gpurun_out/bench_c3.json')); print('c3', round(d['value'],1), d['roofline']['frac'], d['clocks'], d['schedule_realized']['measured_clk_per_trip'])"
timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/bench_c4.json')); print('c4', round(d['value'],1), d['roofline']['frac'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 20 --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
SCHED=fa_fwd timeout 900 ncu --set full --clock-control none --import-source on -k regex:fa_fwd -c 1 -f -o gpurun_out/fa_c3_full python tools/prof_run.py fa 2 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:fa_fwd -c 1 -f -o gpurun_out/fa_c4_full python tools/prof_run.py fa_causal 2 > /dev/null 2>&1
timeout 300 python tools/realized_gantt.py fa_fwd gpurun_out/realized_fa_fwd > /dev/null 2>&1
timeout 300 python tools/gpu_debug.py perf 2>&1 | grep gemm
ls gpurun_out/
