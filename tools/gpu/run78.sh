timeout 900 python bench.py --config c4 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c4_wl.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/bench_c4_wl.json')); print(d['value'], d['fa_bwd']['value'], d['clocks'])"
timeout 600 ncu --set full --clock-control none -k regex:fa_fwd -c 1 -f -o gpurun_out/fa_c4_wl python tools/prof_run.py fa_causal 2 > /dev/null 2>&1
ncu -i gpurun_out/fa_c4_wl.ncu-rep --page details 2>/dev/null | grep -E "L2 Hit Rate|DRAM Throughput|Duration" | head -4
