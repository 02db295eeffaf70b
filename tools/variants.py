"""Time FA C3 for each library variant given on the command line (TWFA_LIB per subprocess)."""
import os, subprocess, sys
code = r'''
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2512_18134_b200 as twfa
from tests import oracle_lib
import numpy as np
_sched = os.environ.get("SCHED", "fa_fwd")
if ":" in _sched:  # problem:solution-path (experiments)
    _pn, _sp = _sched.split(":")
    p = twfa.Plan(twfa.load_schedule(_pn)[0], open(os.path.join(twfa.schedule_dir(), _sp + ".solution.json")).read())
else:
    p = twfa.Plan(*twfa.load_schedule(_sched))
B, H, S = [int(x) for x in os.environ.get("SHAPE", "4,32,8192").split(",")]
causal = os.environ.get("CAUSAL", "0") == "1"
q, k, v = (torch.randn(B, H, S, 128, device="cuda").to(torch.bfloat16) for _ in range(3))
for _ in range(3): twfa.fa_fwd(p, q, k, v, causal=causal)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); n = 20
for _ in range(n): twfa.fa_fwd(p, q, k, v, causal=causal)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n
fl = 4 * B * H * S * S * 128 / (2 if causal else 1)
g = torch.Generator().manual_seed(7)
qs, ks, vs = (torch.randn(1, 2, 512, 128, generator=g).to(torch.bfloat16) for _ in range(3))
o = twfa.fa_fwd(p, qs.cuda(), ks.cuda(), vs.cuda()).float().cpu().numpy()
ro, _ = oracle_lib.attention(qs.float().numpy(), ks.float().numpy(), vs.float().numpy())
print(f"{os.environ.get('SCHED','fa_fwd')} {os.path.basename(os.environ['TWFA_LIB'])}: {ms:.3f} ms {fl/ms/1e9:.1f} TFLOPS  maxerr {np.abs(o-ro).max():.2e}", flush=True)
'''
scheds = os.environ.get("SCHEDS", "fa_fwd").split(",")
reps = int(os.environ.get("REPS", "1"))
for rep in range(reps):  # interleaved repeats: A/B on the same box and thermal state
  for sch in scheds:
    for lib in sys.argv[1:]:
      env = dict(os.environ, TWFA_LIB=os.path.abspath(lib), SCHED=sch)
      r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=120)
      print(r.stdout.strip() or r.stderr[-2000:], flush=True)
