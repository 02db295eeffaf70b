cat > /tmp/g.py <<'PY'
import os, sys, torch, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2512_18134_b200 as twfa
from tests import oracle_lib
gp = twfa.Plan(*twfa.load_schedule("gemm_mainloop"))
M = 8192
a = torch.randn(M, M, device="cuda").to(torch.bfloat16); b = torch.randn(M, M, device="cuda").to(torch.bfloat16)
for _ in range(3): c = twfa.gemm(gp, a, b)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): twfa.gemm(gp, a, b)
e1.record(); torch.cuda.synchronize(); ms = e0.elapsed_time(e1) / 20
ref = (a[:256].float() @ b[:256].float().T)
err = (c[:256, :256].float() - ref[:, :256]).abs().max().item()
print(os.path.basename(os.environ.get("TWFA_LIB", "libtwfa.so")), f"gemm 8192^3 {ms:.3f} ms {2*M**3/ms/1e9:.1f} TFLOPS maxerr {err:.3e}")
PY
for L in paper_2512_18134_b200/libtwfa.so paper_2512_18134_b200/variants/gemm_elect.so; do for i in 1 2; do TWFA_LIB=$L timeout 120 python /tmp/g.py; done; done
