## tools/gpu/run1.sh
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
cat gpurun_out/pytest_gpu.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.txt 2>&1; tail -3 gpurun_out/smoke.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c3.json 2>gpurun_out/bench_c3.err; cat gpurun_out/bench_c3.json; tail -3 gpurun_out/bench_c3.err
timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2>&1; cat gpurun_out/bench_c4.json
timeout 300 python -c "
import torch,time
import torch.nn.functional as F
q,k,v=(torch.randn(4,32,8192,128,device='cuda',dtype=torch.bfloat16) for _ in range(3))
for causal,shape in ((False,(4,32,8192)),(True,(2,32,16384))):
  B,H,S=shape
  q,k,v=(torch.randn(B,H,S,128,device='cuda',dtype=torch.bfloat16) for _ in range(3))
  for _ in range(3): F.scaled_dot_product_attention(q,k,v,is_causal=causal)
  torch.cuda.synchronize()
  e0,e1=torch.cuda.Event(True),torch.cuda.Event(True)
  e0.record()
  for _ in range(10): F.scaled_dot_product_attention(q,k,v,is_causal=causal)
  e1.record(); torch.cuda.synchronize()
  ms=e0.elapsed_time(e1)/10
  fl=4*B*H*S*S*128/(2 if causal else 1)
  print('sdpa causal',causal, ms, fl/ms/1e9,'TFLOPS')
" > gpurun_out/sdpa.txt 2>&1; cat gpurun_out/sdpa.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 20 --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1; tail -3 gpurun_out/ncu_bench.log

## tools/gpu/run2.sh
cd $GRAFT_REPO_ROOT
SCHEDS=fa_fwd,fa_fwd_cal,fa_fwd_tcvl,fa_fwd:experiments/E1_fa4,fa_fwd:experiments/E2_pertile,fa_fwd:experiments/E3_sep timeout 600 python tools/variants.py paper_2512_18134_b200/libtwfa.so > gpurun_out/variants.txt 2>&1
cat gpurun_out/variants.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fa_fwd -c 1 -f -o gpurun_out/fa_c3_full python tools/prof_run.py fa 2 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log

## tools/gpu/run3.sh
timeout 300 python tools/trace_stats.py 4 32 8192 fa_fwd > gpurun_out/trace_c3.txt 2>&1
timeout 300 python tools/trace_stats.py 4 32 8192 fa_fwd_cal >> gpurun_out/trace_c3.txt 2>&1

## tools/gpu/run4.sh
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
V=paper_2512_18134_b200/variants
SCHEDS=fa_fwd,fa_fwd:experiments/E1_fa4,fa_fwd:experiments/E3_sep timeout 900 python tools/variants.py $V/poly1000.so $V/poly8.so $V/poly4.so $V/poly2.so 2>&1

## tools/gpu/run5.sh
export TWFA_LIB=paper_2512_18134_b200/variants/poly1000.so
timeout 300 python tools/trace_stats.py 4 32 8192 fa_fwd:experiments/E1_fa4 > gpurun_out/trace_e1.txt 2>&1
timeout 300 python tools/trace_stats.py 4 32 8192 fa_fwd > gpurun_out/trace_fa2.txt 2>&1

## tools/gpu/run6.sh
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
SCHEDS=fa_fwd,fa_fwd_cal,fa_fwd:experiments/E1_fa4,fa_fwd:experiments/E2_pertile,fa_fwd:experiments/E3_sep timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so 2>&1
timeout 300 python tools/trace_stats.py 4 32 8192 fa_fwd:experiments/E1_fa4 > gpurun_out/trace_e1.txt 2>&1
timeout 300 python tools/trace_stats.py 4 32 8192 fa_fwd > gpurun_out/trace_fa.txt 2>&1

## tools/gpu/run7.sh
SCHED=fa_fwd:experiments/E1_fa4 timeout 900 ncu --set full --clock-control none --import-source on -k regex:fa_fwd -c 1 -f -o gpurun_out/e1_full python tools/prof_run.py fa 2 > gpurun_out/ncu_e1.log 2>&1
tail -2 gpurun_out/ncu_e1.log

## tools/gpu/run8.sh
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
SCHEDS=fa_fwd,fa_fwd_cal,fa_fwd_tcvl,fa_fwd:experiments/E1_fa4,fa_fwd:experiments/E2_pertile,fa_fwd:experiments/E3_sep timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so 2>&1
TWFA_KERNEL=interpreter SCHEDS=fa_fwd,fa_fwd:experiments/E1_fa4 timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so 2>&1
timeout 300 python tools/trace_stats.py 4 32 8192 fa_fwd:experiments/E1_fa4 > gpurun_out/trace_e1.txt 2>&1
timeout 300 python tools/trace_stats.py 4 32 8192 fa_fwd > gpurun_out/trace_fa.txt 2>&1

## tools/gpu/run9.sh
SCHED=fa_fwd timeout 900 ncu --set full --clock-control none --import-source on -k regex:fa_fwd -c 1 -f -o gpurun_out/spec_full python tools/prof_run.py fa 2 > gpurun_out/ncu_spec.log 2>&1
tail -2 gpurun_out/ncu_spec.log

## tools/gpu/run10.sh
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
SCHEDS=fa_fwd,fa_fwd:experiments/E1_fa4 timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so 2>&1
TWFA_KERNEL=interpreter SCHEDS=fa_fwd,fa_fwd:experiments/E1_fa4 timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so 2>&1
timeout 300 python tools/trace_stats.py 4 32 8192 fa_fwd:experiments/E1_fa4 > gpurun_out/trace_e1.txt 2>&1

## tools/gpu/run11.sh
V=paper_2512_18134_b200/variants
SCHEDS=fa_fwd,fa_fwd:experiments/E1_fa4 timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so $V/poly8.so $V/poly4.so $V/poly2.so 2>&1

## tools/gpu/run12.sh
cd tools/calib && for f in ubench ubench_ex ubench_bar; do echo "== $f"; timeout 120 ./$f; done

## tools/gpu/run13.sh
SCHEDS=fa_fwd,fa_fwd_cal,fa_fwd_tcvl,fa_fwd:experiments/E1_fa4,fa_fwd:experiments/E2_pertile,fa_fwd:experiments/E3_sep timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so 2>&1

## tools/gpu/run14.sh
SCHED=fa_fwd_tcvl timeout 900 ncu --set full --clock-control none --import-source on -k regex:fa_fwd -c 1 -f -o gpurun_out/tcvl_full python tools/prof_run.py fa 2 > gpurun_out/ncu_tcvl.log 2>&1
tail -1 gpurun_out/ncu_tcvl.log

## tools/gpu/run15.sh
REPS=3 SCHEDS=fa_fwd_tcvl,fa_fwd:experiments/E1_fa4 timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so paper_2512_18134_b200/variants/defer.so 2>&1

## tools/gpu/run16.sh
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c3.json 2>gpurun_out/bench_c3.err; cat gpurun_out/bench_c3.json
timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2>&1; cat gpurun_out/bench_c4.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 20 --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
SCHED=fa_fwd timeout 900 ncu --set full --clock-control none --import-source on -k regex:fa_fwd -c 1 -f -o gpurun_out/fa_c3_full python tools/prof_run.py fa 2 > /dev/null 2>&1
timeout 300 python tools/trace_stats.py 4 32 8192 fa_fwd > gpurun_out/trace_c3.txt 2>&1

## tools/gpu/run17.sh
REPS=3 SCHEDS=fa_fwd timeout 900 python tools/variants.py paper_2512_18134_b200/variants/nosplits.so paper_2512_18134_b200/variants/splits.so 2>&1

## tools/gpu/run18.sh
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
REPS=2 SCHEDS=fa_fwd,fa_fwd_fixedtc,fa_fwd:experiments/E1_fa4 timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so 2>&1

## tools/gpu/run19.sh
timeout 300 python tools/trace_stats.py 4 32 8192 fa_fwd > gpurun_out/trace_c3.txt 2>&1
timeout 300 python tools/trace_stats.py 2 32 16384 fa_fwd 1 > gpurun_out/trace_c4.txt 2>&1

## tools/gpu/run20.sh
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
cat > /tmp/ring2check.py <<'PY'
import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2512_18134_b200 as twfa
from tests import oracle_lib
p = twfa.Plan(*twfa.load_schedule("fa_fwd_ring2"))
print(p.describe()["kernel"])
for (B, H, S, causal) in [(1, 2, 512, False), (1, 2, 640, True), (2, 1, 300, False), (1, 1, 64, False), (1,1,100,True)]:
    g = torch.Generator().manual_seed(7)
    q, k, v = (torch.randn(B, H, S, 128, generator=g).to(torch.bfloat16) for _ in range(3))
    o, lse = twfa.fa_fwd(p, q.cuda(), k.cuda(), v.cuda(), causal=causal, return_lse=True)
    ro, rl = oracle_lib.attention(q.float().numpy(), k.float().numpy(), v.float().numpy(), causal=causal)
    e = np.abs(o.float().cpu().numpy() - ro)
    print(B, H, S, causal, "max", e.max(), "mean", e.mean(), "lse", np.abs(lse.cpu().numpy() - rl).max(), flush=True)
PY
timeout 300 python /tmp/ring2check.py
REPS=2 SCHEDS=fa_fwd,fa_fwd_ring2 timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so 2>&1

## tools/gpu/run21.sh
REPS=2 SCHEDS=fa_fwd,fa_fwd_ring2,fa_fwd_ring2:experiments/R2_sep,fa_fwd:experiments/E1_fa4 timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so 2>&1
timeout 300 python tools/trace_stats.py 4 32 8192 fa_fwd_ring2:experiments/R2_sep > gpurun_out/trace_r2.txt 2>&1

## tools/gpu/run22.sh
REPS=2 SCHEDS=fa_fwd_ring2:experiments/R2_pertile,fa_fwd:experiments/E2_pertile timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so 2>&1
timeout 300 python tools/trace_stats.py 4 32 8192 fa_fwd_ring2:experiments/R2_pertile > gpurun_out/trace_r2p.txt 2>&1

## tools/gpu/run23.sh
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c3.json 2>gpurun_out/bench_c3.err; cat gpurun_out/bench_c3.json; tail -2 gpurun_out/bench_c3.err
for S in 1024 2048 4096 8192 16384 32768; do
  timeout 600 python bench.py --config c5 --seq $S --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5 S=%d'%d['config']['S'], round(d['value'],1), 'TF/s', round(d['ms_per_step'],3),'ms', 'e2e', round(d['e2e']['value'],1), 'trip', d['schedule_realized']['measured_clk_per_trip'])"
done

## tools/gpu/run24.sh
REPS=3 SCHEDS=fa_fwd,fa_fwd_vlcal timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so 2>&1

## tools/gpu/run25.sh
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), d['roofline']['frac'], d['schedule_realized'], d['config']['schedule'])"
timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4', round(d['value'],1), d['schedule_realized']['measured_clk_per_trip'])"

## tools/gpu/run26.sh
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python tools/calibrate.py > gpurun_out/calibration.json 2>gpurun_out/calibration.err; tail -3 gpurun_out/calibration.err; cat gpurun_out/calibration.json
timeout 300 python tools/realized_gantt.py fa_fwd gpurun_out/realized_fa_fwd 2>&1 | tail -20

## tools/gpu/run27.sh
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
REPS=3 SCHEDS=fa_fwd,fa_fwd_vl,fa_fwd_cal timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so 2>&1
timeout 300 python tools/realized_gantt.py fa_fwd gpurun_out/realized_fa_fwd 2>&1 | tail -3

## tools/gpu/run28.sh
V=paper_2512_18134_b200/variants
REPS=3 SCHEDS=fa_fwd timeout 900 python tools/variants.py $V/poly1000.so $V/poly8.so $V/poly4.so 2>&1

## tools/gpu/run29.sh
cp /tmp/old_order.so paper_2512_18134_b200/variants/old_order.so 2>/dev/null
REPS=3 SCHEDS=fa_fwd timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so paper_2512_18134_b200/variants/poly1000.so 2>&1
timeout 600 python -m pytest tests/test_gpu_trace.py -q 2>&1 | tail -1

## tools/gpu/run30.sh
REPS=3 SCHEDS=fa_fwd timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so paper_2512_18134_b200/variants/solo.so 2>&1

## tools/gpu/run31.sh
REPS=3 CAUSAL=1 SHAPE=2,32,16384 SCHEDS=fa_fwd timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so paper_2512_18134_b200/variants/snake.so 2>&1

## tools/gpu/run32.sh
V=paper_2512_18134_b200/variants
REPS=3 SCHEDS=fa_fwd timeout 900 python tools/variants.py $V/notok.so $V/tok.so 2>&1

## tools/gpu/run33.sh
V=paper_2512_18134_b200/variants
cat > /tmp/chk.py <<'PY'
import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2512_18134_b200 as twfa
from tests import oracle_lib
p = twfa.Plan(*twfa.load_schedule("fa_fwd"))
for (B, H, S, causal) in [(1, 2, 512, False), (1, 2, 640, True), (2, 1, 300, False), (1, 1, 100, True), (3, 2, 1000, False)]:
    g = torch.Generator().manual_seed(7)
    q, k, v = (torch.randn(B, H, S, 128, generator=g).to(torch.bfloat16) for _ in range(3))
    o, lse = twfa.fa_fwd(p, q.cuda(), k.cuda(), v.cuda(), causal=causal, return_lse=True)
    ro, rl = oracle_lib.attention(q.float().numpy(), k.float().numpy(), v.float().numpy(), causal=causal)
    e = np.abs(o.float().cpu().numpy() - ro)
    print(os.path.basename(os.environ["TWFA_LIB"]), B, H, S, causal, "max", e.max(), "mean", e.mean(), flush=True)
PY
TWFA_LIB=$V/tmaepi.so timeout 300 python /tmp/chk.py
REPS=3 SCHEDS=fa_fwd timeout 900 python tools/variants.py $V/stgepi.so $V/tmaepi.so 2>&1
REPS=2 CAUSAL=1 SHAPE=2,32,16384 SCHEDS=fa_fwd timeout 900 python tools/variants.py $V/stgepi.so $V/tmaepi.so 2>&1

## tools/gpu/run34.sh
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c3.json 2>gpurun_out/bench_c3.err; python -c "import json; d=json.load(open('gpurun_out/bench_c3.json')); print('c3', round(d['value'],1), d['roofline']['frac'], d['clocks'], d['schedule_realized']['measured_clk_per_trip'])"
timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/bench_c4.json')); print('c4', round(d['value'],1), d['roofline']['frac'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 20 --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
SCHED=fa_fwd timeout 900 ncu --set full --clock-control none --import-source on -k regex:fa_fwd -c 1 -f -o gpurun_out/fa_c3_full python tools/prof_run.py fa 2 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:fa_fwd -c 1 -f -o gpurun_out/fa_c4_full python tools/prof_run.py fa_causal 2 > /dev/null 2>&1
timeout 300 python tools/realized_gantt.py fa_fwd gpurun_out/realized_fa_fwd > /dev/null 2>&1
timeout 300 python tools/gpu_debug.py perf 2>&1 | grep gemm
ls gpurun_out/

## tools/gpu/run35.sh
timeout 300 python tools/trace_stats.py 4 32 8192 fa_fwd > gpurun_out/trace_c3.txt 2>&1
timeout 300 python tools/trace_stats.py 2 32 16384 fa_fwd 1 > gpurun_out/trace_c4.txt 2>&1

## tools/gpu/run36.sh
sed -i 's/"fa_fwd_ring2"/"fa_fwd_split"/' /tmp/chk2.py 2>/dev/null
cat > /tmp/chk2.py <<'PY'
import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2512_18134_b200 as twfa
from tests import oracle_lib
p = twfa.Plan(*twfa.load_schedule("fa_fwd_split"))
print(p.describe()["kernel"])
for (B, H, S, causal) in [(1, 2, 512, False), (1, 2, 640, True), (2, 1, 300, False), (1, 1, 100, True), (3, 2, 1000, False)]:
    g = torch.Generator().manual_seed(7)
    q, k, v = (torch.randn(B, H, S, 128, generator=g).to(torch.bfloat16) for _ in range(3))
    o, lse = twfa.fa_fwd(p, q.cuda(), k.cuda(), v.cuda(), causal=causal, return_lse=True)
    ro, rl = oracle_lib.attention(q.float().numpy(), k.float().numpy(), v.float().numpy(), causal=causal)
    e = np.abs(o.float().cpu().numpy() - ro)
    print(B, H, S, causal, "max", e.max(), "mean", e.mean(), "lse", np.abs(lse.cpu().numpy() - rl).max(), flush=True)
PY
timeout 300 python /tmp/chk2.py
REPS=3 SCHEDS=fa_fwd,fa_fwd_split timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so 2>&1

## tools/gpu/run37.sh
cat > /tmp/g.py <<'PY'
import os, sys, torch, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2512_18134_b200 as twfa
from tests import oracle_lib
gp = twfa.Plan(*twfa.load_schedule("gemm_mainloop"))
M = 8192
a = torch.randn(M, M, device="cuda").to(torch.bfloat16); b = torch.randn(M, M, device="cuda").to(torch.bfloat16)
for _ in range(3): c = twfa.gemm(gp, a, b)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): twfa.gemm(gp, a, b)
e1.record(); torch.cuda.synchronize(); ms = e0.elapsed_time(e1) / 20
ref = (a[:256].float() @ b[:256].float().T)
err = (c[:256, :256].float() - ref[:, :256]).abs().max().item()
print(os.path.basename(os.environ.get("TWFA_LIB", "libtwfa.so")), f"gemm 8192^3 {ms:.3f} ms {2*M**3/ms/1e9:.1f} TFLOPS maxerr {err:.3e}")
PY
for L in paper_2512_18134_b200/libtwfa.so paper_2512_18134_b200/variants/gemm_elect.so; do for i in 1 2; do TWFA_LIB=$L timeout 120 python /tmp/g.py; done; done

## tools/gpu/run38.sh
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
REPS=3 SCHEDS=fa_fwd timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so 2>&1
REPS=2 CAUSAL=1 SHAPE=2,32,16384 SCHEDS=fa_fwd timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so 2>&1

## tools/gpu/run39.sh
timeout 300 python tools/trace_stats.py 4 32 8192 fa_fwd > gpurun_out/trace39.txt 2>&1
tail -5 gpurun_out/trace39.txt

## tools/gpu/run40.sh
V=paper_2512_18134_b200/variants
REPS=2 SCHEDS=fa_fwd timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so $V/poly2.so $V/poly4.so $V/poly8.so 2>&1
REPS=2 SCHEDS=fa_fwd_fixedtc:experiments/E1_fa4 timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so $V/poly4.so 2>&1

## tools/gpu/run41.sh
V=paper_2512_18134_b200/variants
REPS=2 SCHEDS=fa_fwd timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so $V/whatif1.so $V/whatif2.so $V/whatif3.so 2>&1

## tools/gpu/run42.sh
V=paper_2512_18134_b200/variants
REPS=3 SCHEDS=fa_fwd timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so $V/lean.so 2>&1
REPS=2 CAUSAL=1 SHAPE=2,32,16384 SCHEDS=fa_fwd timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so $V/lean.so 2>&1

## tools/gpu/run43.sh
V=paper_2512_18134_b200/variants
timeout 60 tools/calib/ubench_mmaq
REPS=2 SCHEDS=fa_fwd timeout 900 python tools/variants.py $V/lean.so $V/whatif4.so 2>&1

## tools/gpu/run44.sh
export TWFA_LIB=paper_2512_18134_b200/variants/lean.so
SCHED=fa_fwd timeout 900 ncu --set full --clock-control none --import-source on -k regex:fa_fwd -c 1 -f -o gpurun_out/lean_full python tools/prof_run.py fa 2 > gpurun_out/ncu_lean.log 2>&1
tail -3 gpurun_out/ncu_lean.log

## tools/gpu/run45.sh
V=paper_2512_18134_b200/variants
REPS=2 SCHEDS=fa_fwd,fa_fwd_ring2 timeout 900 python tools/variants.py $V/lean_r2.so 2>&1

## tools/gpu/run46.sh
V=paper_2512_18134_b200/variants
REPS=2 SCHEDS=fa_fwd,fa_fwd_split timeout 900 python tools/variants.py $V/lean_split.so 2>&1

## tools/gpu/run47.sh
V=paper_2512_18134_b200/variants
REPS=2 SCHEDS=fa_fwd timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so $V/parts4.so $V/parts8.so 2>&1
REPS=1 CAUSAL=1 SHAPE=2,32,16384 SCHEDS=fa_fwd timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so $V/parts4.so $V/parts8.so 2>&1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3

## tools/gpu/run48.sh
timeout 300 python tools/gpu/bwd_check.py 2>&1 | tail -20

## tools/gpu/run49.sh
timeout 600 python -m pytest tests/test_gpu_bwd.py -x -q 2>&1 | tail -5

## tools/gpu/run50.sh
V=paper_2512_18134_b200/variants
timeout 600 python tools/gpu/bwd_time.py paper_2512_18134_b200/libtwfa.so $V/bwdw1.so $V/bwdw2.so

## tools/gpu/run51.sh
SHAPE=4,32,8192 timeout 600 python tools/gpu/bwd_time.py paper_2512_18134_b200/variants/bwdprof.so 2>&1 | head -3
cat > /tmp/p.py <<'PY'
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2512_18134_b200 as twfa
fp = twfa.Plan(*twfa.load_schedule("fa_fwd")); bp = twfa.Plan(*twfa.load_schedule(os.environ.get("BSCHED", "fa_bwd")))
B, H, S = 4, 32, 8192
q, k, v, do = (torch.randn(B, H, S, 128, device="cuda").to(torch.bfloat16) for _ in range(4))
o, lse = twfa.fa_fwd(fp, q, k, v, return_lse=True)
twfa.fa_bwd(bp, q, k, v, o, do, lse); torch.cuda.synchronize()
PY
TWFA_LIB=paper_2512_18134_b200/variants/bwdprof.so timeout 300 python /tmp/p.py 2>&1 | grep PROF | sort -k3 -n | head -60

## tools/gpu/run52.sh
timeout 600 python -m pytest tests/test_gpu_bwd.py -x -q 2>&1 | tail -2
timeout 600 python tools/gpu/bwd_time.py paper_2512_18134_b200/libtwfa.so
CAUSAL=1 SHAPE=2,32,16384 timeout 600 python tools/gpu/bwd_time.py paper_2512_18134_b200/libtwfa.so

## tools/gpu/run53.sh
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; tail -c 3000 gpurun_out/bench_c3.json

## tools/gpu/run54.sh
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fa_bwd_kernel -c 1 -f -o gpurun_out/bwd_c3_full python tools/prof_run.py bwd 2 > gpurun_out/ncu_bwd.log 2>&1; tail -2 gpurun_out/ncu_bwd.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_bwd.csv python tools/prof_run.py bwd 3 > /dev/null 2>&1
timeout 900 python bench.py --config c4 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; tail -c 600 gpurun_out/bench_c4.json

## tools/gpu/run55.sh
for S in 1024 2048 4096 8192 16384 32768; do
  timeout 600 python bench.py --config c5 --seq $S --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c5_$S.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/c5_$S.json')); print($S, round(d['value'],1), round(d['ms_per_step'],3), round(d['e2e']['value'],1), round(d['fa_bwd']['value'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 2>&1 | tail -c 800

## tools/gpu/run56.sh
V=paper_2512_18134_b200/variants
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
REPS=3 SCHEDS=fa_fwd timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so $V/nospec.so 2>&1
REPS=2 CAUSAL=1 SHAPE=2,32,16384 SCHEDS=fa_fwd timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so $V/nospec.so 2>&1

## tools/gpu/run57.sh
timeout 600 python -m pytest tests/test_gpu_bwd.py -x -q 2>&1 | tail -2
timeout 600 python tools/gpu/bwd_time.py paper_2512_18134_b200/libtwfa.so
BSCHED=fa_bwd_regp timeout 600 python tools/gpu/bwd_time.py paper_2512_18134_b200/libtwfa.so
CAUSAL=1 SHAPE=2,32,16384 timeout 600 python tools/gpu/bwd_time.py paper_2512_18134_b200/libtwfa.so

## tools/gpu/run58.sh
timeout 120 python -m pytest tests/test_gpu_bwd.py -x -q 2>&1 | tail -3
timeout 120 python tools/gpu/bwd_time.py paper_2512_18134_b200/libtwfa.so
BSCHED=fa_bwd_regp timeout 120 python tools/gpu/bwd_time.py paper_2512_18134_b200/libtwfa.so
CAUSAL=1 SHAPE=2,32,16384 timeout 120 python tools/gpu/bwd_time.py paper_2512_18134_b200/libtwfa.so

## tools/gpu/run59.sh
timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 120 python tools/gpu/bwd_time.py paper_2512_18134_b200/libtwfa.so
BSCHED=fa_bwd_split timeout 120 python tools/gpu/bwd_time.py paper_2512_18134_b200/libtwfa.so

## tools/gpu/run60.sh
V=paper_2512_18134_b200/variants
timeout 120 python tools/gpu/bwd_time.py paper_2512_18134_b200/libtwfa.so $V/bwdred.so
BSCHED=fa_bwd_split timeout 120 python tools/gpu/bwd_time.py paper_2512_18134_b200/libtwfa.so $V/bwdred.so
TWFA_LIB=$V/bwdred.so timeout 120 python -m pytest tests/test_gpu_bwd.py -x -q 2>&1 | tail -1

## tools/gpu/run61.sh
SCHED=fa_fwd timeout 900 ncu --set full --clock-control none --import-source on -k regex:fa_fwd -c 1 -f -o gpurun_out/spec_ex_full python tools/prof_run.py fa 2 > gpurun_out/ncu_specex.log 2>&1
tail -1 gpurun_out/ncu_specex.log

## tools/gpu/run62.sh
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
sed -n '1,17p' tools/gpu/run37.sh > /tmp/g.sh
bash /tmp/g.sh
for L in paper_2512_18134_b200/libtwfa.so paper_2512_18134_b200/variants/gemm_old.so paper_2512_18134_b200/libtwfa.so paper_2512_18134_b200/variants/gemm_old.so; do TWFA_LIB=$L timeout 120 python /tmp/g.py; done

## tools/gpu/run63.sh
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; tail -c 400 gpurun_out/bench_final.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; grep -c fa_fwd_spec gpurun_out/launches_final.csv

## tools/gpu/run64.sh
timeout 600 compute-sanitizer --tool memcheck --print-limit 10 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer_memcheck.txt 2>&1; tail -5 gpurun_out/sanitizer_memcheck.txt
timeout 600 compute-sanitizer --tool racecheck --print-limit 10 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer_racecheck.txt 2>&1; tail -5 gpurun_out/sanitizer_racecheck.txt

## tools/gpu/run65.sh
V=paper_2512_18134_b200/variants
timeout 300 python -m pytest tests/test_gpu_fa.py tests/test_gpu_trace.py -x -q 2>&1 | tail -1
REPS=3 SCHEDS=fa_fwd timeout 600 python tools/variants.py paper_2512_18134_b200/libtwfa.so $V/noxtile.so 2>&1
REPS=2 CAUSAL=1 SHAPE=2,32,16384 SCHEDS=fa_fwd timeout 600 python tools/variants.py paper_2512_18134_b200/libtwfa.so $V/noxtile.so 2>&1

## tools/gpu/run66.sh
V=paper_2512_18134_b200/variants
REPS=2 SCHEDS=fa_fwd timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so $V/poly16.so $V/poly8.so $V/poly4.so $V/parts2.so $V/parts8.so 2>&1

## tools/gpu/run67.sh
timeout 200 python -m pytest tests/test_gpu_bwd.py -x -q 2>&1 | tail -1
timeout 120 python tools/gpu/bwd_time.py paper_2512_18134_b200/libtwfa.so
timeout 120 python tools/gpu/bwd_time.py paper_2512_18134_b200/libtwfa.so
CAUSAL=1 SHAPE=2,32,16384 timeout 120 python tools/gpu/bwd_time.py paper_2512_18134_b200/libtwfa.so

## tools/gpu/run68.sh
timeout 300 python -m pytest tests/test_gpu_fa.py -x -q -k "cross_tile or many_work" 2>&1 | tail -2

## tools/gpu/run69.sh
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_tile.json 2> gpurun_out/bench_tile.err; python -c "import json; d=json.load(open('gpurun_out/bench_tile.json')); print(d['value'], d['schedule_realized'], d['clocks'])"; tail -3 gpurun_out/bench_tile.err

## tools/gpu/run70.sh
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1

## tools/gpu/run71.sh
timeout 200 python -m pytest tests/test_gpu_bwd.py -x -q 2>&1 | tail -1
for i in 1 2; do timeout 120 python tools/gpu/bwd_time.py paper_2512_18134_b200/libtwfa.so paper_2512_18134_b200/variants/bwd_eager.so; done
BSCHED=fa_bwd_split timeout 120 python tools/gpu/bwd_time.py paper_2512_18134_b200/libtwfa.so paper_2512_18134_b200/variants/bwd_eager.so
CAUSAL=1 SHAPE=2,32,16384 timeout 120 python tools/gpu/bwd_time.py paper_2512_18134_b200/libtwfa.so paper_2512_18134_b200/variants/bwd_eager.so

## tools/gpu/run72.sh
timeout 900 python bench.py --config c4 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c4_final.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/bench_c4_final.json')); print(d['value'], d['fa_bwd']['value'], d['clocks'], d['e2e']['value'])"

## tools/gpu/run73.sh
V=paper_2512_18134_b200/variants
timeout 200 python -m pytest tests/test_gpu_bwd.py -x -q 2>&1 | tail -1
timeout 120 python tools/gpu/bwd_time.py paper_2512_18134_b200/libtwfa.so $V/rd_old.so paper_2512_18134_b200/libtwfa.so $V/rd_old.so
BSCHED=fa_bwd_split timeout 120 python tools/gpu/bwd_time.py paper_2512_18134_b200/libtwfa.so $V/rd_old.so

## tools/gpu/run74.sh
V=paper_2512_18134_b200/variants
TWFA_LIB=$V/shalves.so timeout 300 python -m pytest tests/test_gpu_fa.py -x -q -k "not split and not double and not interpreter and not pybind and not host_tool" 2>&1 | tail -1
REPS=3 SCHEDS=fa_fwd timeout 600 python tools/variants.py paper_2512_18134_b200/libtwfa.so $V/shalves.so 2>&1
REPS=2 CAUSAL=1 SHAPE=2,32,16384 SCHEDS=fa_fwd timeout 600 python tools/variants.py paper_2512_18134_b200/libtwfa.so $V/shalves.so 2>&1

## tools/gpu/run75.sh
V=paper_2512_18134_b200/variants
TWFA_LIB=$V/pred.so timeout 300 python -m pytest tests/test_gpu_fa.py -x -q -k "noncausal or causal_matches or ragged or many_work" 2>&1 | tail -1
REPS=3 SCHEDS=fa_fwd timeout 600 python tools/variants.py paper_2512_18134_b200/libtwfa.so $V/pred.so 2>&1

## tools/gpu/run76.sh
timeout 300 python -m pytest tests/test_gpu_fa.py -x -q -k "causal or ragged or many_work or cross_tile or cudnn" 2>&1 | tail -1
for i in 1 2; do
CAUSAL=1 SHAPE=2,32,16384 SCHEDS=fa_fwd timeout 600 python tools/variants.py paper_2512_18134_b200/libtwfa.so 2>&1
TWFA_WORK_LISTS=0 CAUSAL=1 SHAPE=2,32,16384 SCHEDS=fa_fwd timeout 600 python tools/variants.py paper_2512_18134_b200/libtwfa.so 2>&1 | sed 's/^/nolist /'
done

## tools/gpu/run77.sh
timeout 300 python -m pytest tests/test_gpu_fa.py tests/test_gpu_bwd.py -x -q -k "causal or ragged or many_work or cross_tile or tail or split" 2>&1 | tail -1
for i in 1 2; do
CAUSAL=1 SHAPE=2,32,16384 timeout 120 python tools/gpu/bwd_time.py paper_2512_18134_b200/libtwfa.so
TWFA_WORK_LISTS=0 CAUSAL=1 SHAPE=2,32,16384 timeout 120 python tools/gpu/bwd_time.py paper_2512_18134_b200/libtwfa.so | sed 's/^/nolist /'
done
CAUSAL=1 SHAPE=2,32,16384 SCHEDS=fa_fwd timeout 600 python tools/variants.py paper_2512_18134_b200/libtwfa.so 2>&1

## tools/gpu/run78.sh
timeout 900 python bench.py --config c4 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c4_wl.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/bench_c4_wl.json')); print(d['value'], d['fa_bwd']['value'], d['clocks'])"
timeout 600 ncu --set full --clock-control none -k regex:fa_fwd -c 1 -f -o gpurun_out/fa_c4_wl python tools/prof_run.py fa_causal 2 > /dev/null 2>&1
ncu -i gpurun_out/fa_c4_wl.ncu-rep --page details 2>/dev/null | grep -E "L2 Hit Rate|DRAM Throughput|Duration" | head -4

## tools/gpu/run79.sh
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err; python -c "import json; d=json.load(open('gpurun_out/bench_e2e.json')); print(d['value'], d['e2e'])"; tail -3 gpurun_out/bench_e2e.err

## tools/gpu/run80.sh
timeout 600 ncu --set full --clock-control none -k regex:gemm -c 1 -f -o gpurun_out/gemm_full python tools/prof_run.py gemm 2 > /dev/null 2>&1
ncu -i gpurun_out/gemm_full.ncu-rep --page details 2>/dev/null | grep -E "Duration|SM Frequency|L2 Hit Rate|DRAM Throughput|Memory Throughput|L1/TEX Hit|Compute \(SM\) Throughput" | head -10

## tools/gpu/run81.sh
timeout 200 python -m pytest tests/test_gpu_bwd.py -x -q 2>&1 | tail -1
for B in fa_bwd fa_bwd_qstage fa_bwd_split; do BSCHED=$B timeout 120 python tools/gpu/bwd_time.py paper_2512_18134_b200/libtwfa.so | sed "s/^/$B /"; done
for B in fa_bwd fa_bwd_qstage; do BSCHED=$B CAUSAL=1 SHAPE=2,32,16384 timeout 120 python tools/gpu/bwd_time.py paper_2512_18134_b200/libtwfa.so | sed "s/^/$B /"; done

## tools/gpu/run82.sh
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_final2.json 2> gpurun_out/bench_final2.err; python -c "import json; d=json.load(open('gpurun_out/bench_final2.json')); print(d['value'], d['roofline']['frac'], d['clocks'], d['e2e']['value'], d['fa_bwd']['value'], d['cpu_baseline']['value'])"

## tools/gpu/run83.sh
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -c 300
echo
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29556 bench.py --impl reference --gpus 1 --steps 2 --warmup 3 2>/dev/null | tail -c 200

## tools/gpu/run84.sh
V=paper_2512_18134_b200/variants
TWFA_LIB=$V/eager.so timeout 300 python -m pytest tests/test_gpu_fa.py -x -q -k "noncausal or causal_matches or many_work" 2>&1 | tail -1
REPS=3 SCHEDS=fa_fwd timeout 600 python tools/variants.py paper_2512_18134_b200/libtwfa.so $V/eager.so 2>&1
REPS=2 CAUSAL=1 SHAPE=2,32,16384 SCHEDS=fa_fwd timeout 600 python tools/variants.py paper_2512_18134_b200/libtwfa.so $V/eager.so 2>&1

## tools/gpu/run85.sh
for MB in 16 32 48 96; do
TWFA_WL_GROUP_MB=$MB CAUSAL=1 SHAPE=2,32,16384 SCHEDS=fa_fwd timeout 300 python tools/variants.py paper_2512_18134_b200/libtwfa.so 2>&1 | sed "s/^/fwd MB=$MB /"
TWFA_WL_GROUP_MB=$MB CAUSAL=1 SHAPE=2,32,16384 timeout 120 python tools/gpu/bwd_time.py paper_2512_18134_b200/libtwfa.so | sed "s/^/bwd MB=$MB /"
done

## tools/gpu/run86.sh
timeout 120 python tools/gpu/bwd_time.py paper_2512_18134_b200/libtwfa.so paper_2512_18134_b200/variants/bwdw2.so paper_2512_18134_b200/libtwfa.so paper_2512_18134_b200/variants/bwdw2.so

