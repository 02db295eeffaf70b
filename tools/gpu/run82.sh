timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_final2.json 2> gpurun_out/bench_final2.err; python -c "import json; d=json.load(open('gpurun_out/bench_final2.json')); print(d['value'], d['roofline']['frac'], d['clocks'], d['e2e']['value'], d['fa_bwd']['value'], d['cpu_baseline']['value'])"
