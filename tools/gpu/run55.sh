for S in 1024 2048 4096 8192 16384 32768; do
  timeout 600 python bench.py --config c5 --seq $S --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c5_$S.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/c5_$S.json')); print($S, round(d['value'],1), round(d['ms_per_step'],3), round(d['e2e']['value'],1), round(d['fa_bwd']['value'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 2>&1 | tail -c 800
