"""Phases of the fused speculative MX + EX on CTA 0 (diagnostic build with
TWFA_TRACE_SUB=1, TWFA_LIB=<that build>): S ready -> row max / handoff done ->
last exponential issued -> done, medians per softmax warp, C3 shape."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2512_18134_b200 as twfa
prob, sol = twfa.load_schedule("fa_fwd")
plan = twfa.Plan(prob, sol)
ids = [n["id"] for n in json.loads(prob)["graph"]["nodes"]]
nw, cap = 16, 8192
tr = torch.zeros(nw * cap * 8, dtype=torch.int32, device="cuda")
q, k, v = (torch.randn(4, 32, 8192, 128, device="cuda").to(torch.bfloat16) for _ in range(3))
twfa.fa_fwd(plan, q, k, v)
twfa.fa_fwd(plan, q, k, v, trace=tr, trace_cap=cap)
torch.cuda.synchronize()
t = tr.cpu().numpy().view(np.uint32).reshape(nw, cap, 8).astype(np.int64)
d = lambda a, b: (b - a) % (1 << 32)
print("pair" if plan.describe().get("cta_pair") else "single")
for w in range(4, 12):
    rs = [t[w, 1 + i] for i in range(int(t[w, 0, 0])) if ids[t[w, 1 + i, 0]].startswith("MX")]
    rs = rs[len(rs) // 4:]
    a = np.array([[d(r[4], r[6]), d(r[6], r[7]), d(r[7], r[5])] for r in rs])
    print(f"warp {w:2d}: ready->max/handoff {np.median(a[:, 0]):6.0f}  ->last exp {np.median(a[:, 1]):6.0f}  "
          f"->done {np.median(a[:, 2]):6.0f}  total {np.median(a.sum(1)):6.0f}")
