"""Quick first-light checks on the GPU box (prints, never asserts)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2512_18134_b200 as twfa
from tests import oracle_lib
dev = torch.device("cuda:0")
print(torch.cuda.get_device_name(0), flush=True)
what = sys.argv[1] if len(sys.argv) > 1 else "all"
if what in ("all", "gemm"):
    gp = twfa.Plan(*twfa.load_schedule("gemm_mainloop"))
    for (M, N, K) in [(128, 256, 64), (256, 512, 256)]:
        g = torch.Generator().manual_seed(1)
        a = (torch.randn(M, K, generator=g) / 8).to(torch.bfloat16); b = torch.randn(N, K, generator=g).to(torch.bfloat16)
        c = twfa.gemm(gp, a.to(dev), b.to(dev)); torch.cuda.synchronize()
        ref = oracle_lib.gemm_tn(a.float().numpy(), b.float().numpy())
        cc = c.float().cpu().numpy()
        print("gemm", M, N, K, "maxerr", np.abs(cc - ref).max(), "refmax", np.abs(ref).max(), flush=True)
        if np.abs(cc - ref).max() > 0.1:
            print(" c[0,:8]", cc[0, :8], "\n ref[0,:8]", ref[0, :8], flush=True)
if what in ("all", "fa"):
    p = twfa.Plan(*twfa.load_schedule("fa_fwd"))
    for (B, H, S, causal) in [(1, 1, 128, False), (1, 2, 512, False), (1, 2, 512, True)]:
        g = torch.Generator().manual_seed(7)
        q, k, v = (torch.randn(B, H, S, 128, generator=g).to(torch.bfloat16) for _ in range(3))
        o, lse = twfa.fa_fwd(p, q.to(dev), k.to(dev), v.to(dev), causal=causal, return_lse=True)
        torch.cuda.synchronize()
        ro, rl = oracle_lib.attention(q.float().numpy(), k.float().numpy(), v.float().numpy(), causal=causal)
        oo = o.float().cpu().numpy()
        print("fa", B, H, S, causal, "maxerr", np.abs(oo - ro).max(), "mean", np.abs(oo - ro).mean(),
              "lse", np.abs(lse.cpu().numpy() - rl).max(), flush=True)
        if np.abs(oo - ro).max() > 0.1:
            print(" o[0,0,0,:6]", oo[0, 0, 0, :6], "\n ref", ro[0, 0, 0, :6], flush=True)
            print(" lse", lse.cpu().numpy()[0, 0, :4], rl[0, 0, :4], flush=True)
if what in ("all", "perf"):
    p = twfa.Plan(*twfa.load_schedule("fa_fwd"))
    B, H, S = 4, 32, 8192
    q, k, v = (torch.randn(B, H, S, 128, device=dev).to(torch.bfloat16) for _ in range(3))
    for _ in range(3): twfa.fa_fwd(p, q, k, v)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); n = 10
    for _ in range(n): twfa.fa_fwd(p, q, k, v)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(f"fa C3 {ms:.3f} ms  {4*B*H*S*S*128/ms/1e9:.1f} TFLOPS", flush=True)
    e0.record()
    for _ in range(n): torch.nn.functional.scaled_dot_product_attention(q, k, v)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(f"sdpa C3 {ms:.3f} ms  {4*B*H*S*S*128/ms/1e9:.1f} TFLOPS", flush=True)
    gp = twfa.Plan(*twfa.load_schedule("gemm_mainloop"))
    M = 8192
    a = torch.randn(M, M, device=dev).to(torch.bfloat16); b = torch.randn(M, M, device=dev).to(torch.bfloat16)
    for _ in range(3): twfa.gemm(gp, a, b)
    torch.cuda.synchronize(); e0.record()
    for _ in range(n): twfa.gemm(gp, a, b)
    e1.record(); torch.cuda.synchronize(); ms = e0.elapsed_time(e1) / n
    print(f"gemm 8192^3 {ms:.3f} ms {2*M**3/ms/1e9:.1f} TFLOPS", flush=True)
