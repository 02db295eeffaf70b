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
