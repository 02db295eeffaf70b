"""Observed parity errors of the GPU kernels (for setting the test
tolerances at ~3x observed): forward vs the fp64-accumulated oracle, the
backward vs its oracle, and the C3 / C4 shapes against torch SDPA."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2512_18134_b200 as twfa
from tests import oracle_lib
p = twfa.Plan(*twfa.load_schedule("fa_fwd")); bp = twfa.Plan(*twfa.load_schedule("fa_bwd"))
mx = {"o_max": 0, "o_mean": 0, "lse": 0, "bwd_max": 0, "bwd_mean": 0}
for seed, (B, H, S, causal) in enumerate([(1, 2, 512, False), (1, 2, 1024, True), (2, 1, 300, False), (2, 3, 640, True),
                                           (1, 2, 2048, False)]):
    g = torch.Generator().manual_seed(100 + seed)
    q, k, v = (torch.randn(B, H, S, 128, generator=g).to(torch.bfloat16) for _ in range(3))
    o, lse = twfa.fa_fwd(p, q.cuda(), k.cuda(), v.cuda(), causal=causal, return_lse=True)
    ro, rl = oracle_lib.attention(q.float().numpy(), k.float().numpy(), v.float().numpy(), causal=causal)
    e = np.abs(o.float().cpu().numpy() - ro); le = np.abs(lse.cpu().numpy() - rl)
    mx["o_max"] = max(mx["o_max"], e.max()); mx["o_mean"] = max(mx["o_mean"], e.mean()); mx["lse"] = max(mx["lse"], le.max())
    do = torch.randn(B, H, S, 128, generator=g).to(torch.bfloat16)
    dq, dk, dv = twfa.fa_bwd(bp, q.cuda(), k.cuda(), v.cuda(), o, do.cuda(), lse, causal=causal)
    refs = oracle_lib.attention_bwd(q.float().numpy(), k.float().numpy(), v.float().numpy(), o.float().cpu().numpy(),
                                    do.float().numpy(), lse.cpu().numpy(), causal=causal)
    for got, r in zip((dq, dk, dv), refs):
        d = np.abs(got.float().cpu().numpy() - r) / np.abs(r).max()
        mx["bwd_max"] = max(mx["bwd_max"], d.max()); mx["bwd_mean"] = max(mx["bwd_mean"], d.mean())
print("oracle:", {k: float(f"{v:.3e}") for k, v in mx.items()})
for B, H, S, causal, seed in [(4, 32, 8192, False, 2026), (2, 32, 16384, True, 2027)]:
    gd = torch.Generator(device="cuda").manual_seed(seed)
    q, k, v = (torch.randn(B, H, S, 128, device="cuda", generator=gd).to(torch.bfloat16) for _ in range(3))
    o = twfa.fa_fwd(p, q, k, v, causal=causal)
    ref = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=causal)
    d = (o.float() - ref.float()).abs()
    print(f"sdpa B={B} H={H} S={S} causal={causal}: max {d.max().item():.3e} mean {d.mean().item():.3e}")
