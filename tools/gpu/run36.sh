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
