"""Quick GPU check of the FA backward against the C oracle (debug driver)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2512_18134_b200 as twfa
from tests import oracle_lib as ol
fp = twfa.Plan(*twfa.load_schedule("fa_fwd"))
bp = twfa.Plan(*twfa.load_schedule("fa_bwd"))
for (B, H, S, causal) in [(1, 1, 128, False), (1, 2, 256, False), (1, 2, 384, True), (1, 1, 200, False), (1, 2, 320, True)]:
    g = torch.Generator().manual_seed(11)
    q, k, v, do = (torch.randn(B, H, S, 128, generator=g).to(torch.bfloat16) for _ in range(4))
    o, lse = twfa.fa_fwd(fp, q.cuda(), k.cuda(), v.cuda(), causal=causal, return_lse=True)
    t0 = time.time()
    dq, dk, dv = twfa.fa_bwd(bp, q.cuda(), k.cuda(), v.cuda(), o, do.cuda(), lse, causal=causal)
    torch.cuda.synchronize()
    rq, rk, rv = ol.attention_bwd(q.float().numpy(), k.float().numpy(), v.float().numpy(), o.float().cpu().numpy(),
                                  do.float().numpy(), lse.cpu().numpy(), causal=causal)
    out = []
    for name, a, r in (("dq", dq, rq), ("dk", dk, rk), ("dv", dv, rv)):
        a = a.float().cpu().numpy()
        out.append(f"{name} max {np.abs(a - r).max():.3e} rel {np.abs(a - r).max() / np.abs(r).max():.3e}")
    print(B, H, S, causal, " | ".join(out), flush=True)
# timing at the forward's headline shapes
import torch.nn.functional as F
for (B, H, S, causal) in [(4, 32, 8192, False), (2, 32, 16384, True)]:
    q, k, v, do = (torch.randn(B, H, S, 128, device="cuda").to(torch.bfloat16) for _ in range(4))
    o, lse = twfa.fa_fwd(fp, q, k, v, causal=causal, return_lse=True)
    ws = torch.empty(B * H * S * 129 * 4, device="cuda", dtype=torch.uint8)
    for _ in range(2): twfa.fa_bwd(bp, q, k, v, o, do, lse, causal=causal, workspace=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): twfa.fa_bwd(bp, q, k, v, o, do, lse, causal=causal, workspace=ws)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    fl = 10 * B * H * S * S * 128 / (2 if causal else 1)
    # comparator: torch SDPA backward (cuDNN / flash) on the same box
    qr, kr, vr = (t.detach().clone().requires_grad_() for t in (q, k, v))
    with torch.nn.attention.sdpa_kernel([torch.nn.attention.SDPBackend.CUDNN_ATTENTION]):
        out = F.scaled_dot_product_attention(qr, kr, vr, is_causal=causal)
        for _ in range(2): torch.autograd.grad(out, (qr, kr, vr), do, retain_graph=True)
        torch.cuda.synchronize(); e0.record()
        for _ in range(5): torch.autograd.grad(out, (qr, kr, vr), do, retain_graph=True)
        e1.record(); torch.cuda.synchronize()
    ms_ref = e0.elapsed_time(e1) / 5
    print(f"bwd B={B} H={H} S={S} causal={causal}: {ms:.3f} ms {fl / ms / 1e9:.1f} TFLOPS | cuDNN SDPA bwd {ms_ref:.3f} ms {fl / ms_ref / 1e9:.1f}", flush=True)
