"""GEMM 8192^3 (C2) timing per raster group (TWFA_GEMM_GROUP) next to torch.matmul,
20 launches each, CUDA events on the launching stream."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_18134_b200 as twfa
p = twfa.Plan(*twfa.load_schedule("gemm_mainloop"))
M = N = K = 8192
g = torch.Generator(device="cuda").manual_seed(1234)
a = (torch.randn(M, K, device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
b = torch.randn(N, K, device="cuda", generator=g).to(torch.bfloat16)
c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
def t(fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n
fl = 2 * M * N * K
for grp in sys.argv[1:] or ["8"]:
    os.environ["TWFA_GEMM_GROUP"] = grp
    ms = t(lambda: twfa.gemm(p, a, b, out=c))
    err = (c.float() - (a @ b.t()).float()).abs().max().item()
    print(f"group {grp}: {ms:.3f} ms {fl / ms / 1e9:.1f} TFLOPS maxerr {err:.2e}", flush=True)
ms = t(lambda: torch.matmul(a, b.t(), out=c))
print(f"torch.matmul: {ms:.3f} ms {fl / ms / 1e9:.1f} TFLOPS", flush=True)
