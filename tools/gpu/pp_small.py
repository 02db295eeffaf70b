import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, paper_2512_18134_b200 as t
fp=t.Plan(*t.load_schedule('fa_fwd')); bp=t.Plan(*t.load_schedule('fa_bwd_pp'))
q,k,v,do=(torch.randn(1,2,384,128,device='cuda').to(torch.bfloat16) for _ in range(4))
o,lse=t.fa_fwd(fp,q,k,v,causal=True,return_lse=True)
dq,dk,dv=t.fa_bwd(bp,q,k,v,o,do,lse,causal=True)
torch.cuda.synchronize(); print("pp ok", float(dq.float().abs().sum()))
