import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2512_18134_b200 as twfa
from tests import oracle_lib
plan = twfa.Plan(*twfa.load_schedule("fa_fwd"))
def inputs(B,H,S,seed):
    g = torch.Generator(device="cpu").manual_seed(seed)
    return [torch.randn(B, H, S, 128, generator=g).to(torch.bfloat16) for _ in range(3)]
for mag in (1.0, 1.57, 2.0):
  for pair in ("1","0"):
    os.environ["TWFA_PAIR"]=pair
    q,k,v=(x*mag for x in inputs(1,3,514,2013)); q,k,v=(x.to(torch.bfloat16) for x in (q,k,v))
    o,l=twfa.fa_fwd(plan,q.cuda(),k.cuda(),v.cuda(),return_lse=True); torch.cuda.synchronize()
    ro,rl=oracle_lib.attention(q.float().numpy(),k.float().numpy(),v.float().numpy(),causal=False,scale=None)
    of=o.float().cpu().numpy(); m=max(1,np.abs(ro).max()); e=np.abs(of-ro)/m
    idx=np.unravel_index(e.argmax(), e.shape)
    # reference with bf16-rounded P: emulate
    print(f"mag {mag} pair {pair}: max {e.max():.2e} mean {e.mean():.2e} at {idx} maxO {np.abs(ro).max():.2f} maxV {np.abs(v.float().numpy()).max():.2f}")
