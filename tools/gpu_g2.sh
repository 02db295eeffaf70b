# round 2: GPU tests, new default bench (C5 S=8192 strong), 2-rank functional run, ncu of the bench launch
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/g2_bench_n1.json 2> gpurun_out/g2_bench_n1.err; tail -c 600 gpurun_out/g2_bench_n1.err
timeout 600 python bench.py --gpus 2 --share-gpu --steps 5 --warmup 3 --skip-legs --no-cpu-baseline > gpurun_out/g2_bench_n2share.json 2> gpurun_out/g2_bench_n2share.err; tail -c 1500 gpurun_out/g2_bench_n2share.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/g2_ref.json 2> gpurun_out/g2_ref.err
python - <<'PY'
import json
a=json.loads(open('gpurun_out/g2_bench_n1.json').read().strip().splitlines()[-1])
b=json.loads(open('gpurun_out/g2_bench_n2share.json').read().strip().splitlines()[-1])
print("N1", a['value'], a['clocks'], a['job_checksum']['digest'], a['tensor_pipe'])
print("N2share", b['value'], b['job_checksum']['digest'], b['config']['pairs_per_rank'])
print("legs", a.get('legs'))
print("bwd", a.get('fa_bwd',{}).get('value'), "e2e", a.get('e2e',{}).get('value'), a.get('schedule_realized'))
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:fa_fwd --csv --log-file gpurun_out/g2_launches_c5.csv python bench.py --steps 3 --warmup 3 --skip-legs --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fa_fwd_spec -s 3 -c 1 -o gpurun_out/g2_fa_c5_full python bench.py --steps 1 --warmup 3 --skip-legs --no-cpu-baseline > gpurun_out/g2_ncu.log 2>&1; tail -3 gpurun_out/g2_ncu.log
