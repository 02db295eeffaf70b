timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -8
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/g4_bench.json 2> gpurun_out/g4_bench.err; tail -c 400 gpurun_out/g4_bench.err
python - <<'PY'
import json
a=json.loads(open('gpurun_out/g4_bench.json').read().strip().splitlines()[-1])
print(a['value'], a['clocks'], a.get('e2e'), a.get('fa_bwd',{}).get('value'))
PY
