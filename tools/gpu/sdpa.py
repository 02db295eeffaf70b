import torch, torch.nn.functional as F
for causal,(B,H,S) in ((False,(4,32,8192)),):
  q,k,v=(torch.randn(B,H,S,128,device='cuda',dtype=torch.bfloat16) for _ in range(3))
  for _ in range(3): F.scaled_dot_product_attention(q,k,v,is_causal=causal)
  torch.cuda.synchronize()
  e0,e1=torch.cuda.Event(True),torch.cuda.Event(True)
  e0.record()
  for _ in range(20): F.scaled_dot_product_attention(q,k,v,is_causal=causal)
  e1.record(); torch.cuda.synchronize()
  ms=e0.elapsed_time(e1)/20
  print('sdpa causal',causal, ms, 4*B*H*S*S*128/(2 if causal else 1)/ms/1e9,'TFLOPS')
