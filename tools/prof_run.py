"""Tiny driver for ncu captures: warm-up launches then a few profiled ones."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_18134_b200 as twfa
what = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
dev = torch.device("cuda:0")
if what in ("fa", "fa_causal"):
    sched = os.environ.get("SCHED", "fa_fwd")
    if ":" in sched:  # problem:solution-path (experiments)
        pn, sp = sched.split(":")
        p = twfa.Plan(twfa.load_schedule(pn)[0], open(os.path.join(twfa.schedule_dir(), sp + ".solution.json")).read())
    else:
        p = twfa.Plan(*twfa.load_schedule(sched))
    B, H, S = (4, 32, 8192) if what == "fa" else (2, 32, 16384)
    q, k, v = (torch.randn(B, H, S, 128, device=dev).to(torch.bfloat16) for _ in range(3))
    for _ in range(n):
        twfa.fa_fwd(p, q, k, v, causal=(what == "fa_causal"))
elif what in ("bwd", "bwd_causal"):
    fp = twfa.Plan(*twfa.load_schedule("fa_fwd"))
    bp = twfa.Plan(*twfa.load_schedule("fa_bwd"))
    B, H, S = (4, 32, 8192) if what == "bwd" else (2, 32, 16384)
    c = what == "bwd_causal"
    q, k, v, do = (torch.randn(B, H, S, 128, device=dev).to(torch.bfloat16) for _ in range(4))
    o, lse = twfa.fa_fwd(fp, q, k, v, causal=c, return_lse=True)
    for _ in range(n):
        twfa.fa_bwd(bp, q, k, v, o, do, lse, causal=c)
elif what == "gemm":
    p = twfa.Plan(*twfa.load_schedule("gemm_mainloop"))
    a = torch.randn(8192, 8192, device=dev).to(torch.bfloat16)
    b = torch.randn(8192, 8192, device=dev).to(torch.bfloat16)
    for _ in range(n):
        twfa.gemm(p, a, b)
torch.cuda.synchronize()
