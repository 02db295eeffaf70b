SHAPE=4,32,8192 timeout 600 python tools/gpu/bwd_time.py paper_2512_18134_b200/variants/bwdprof.so 2>&1 | head -3
cat > /tmp/p.py <<'PY'
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2512_18134_b200 as twfa
fp = twfa.Plan(*twfa.load_schedule("fa_fwd")); bp = twfa.Plan(*twfa.load_schedule(os.environ.get("BSCHED", "fa_bwd")))
B, H, S = 4, 32, 8192
q, k, v, do = (torch.randn(B, H, S, 128, device="cuda").to(torch.bfloat16) for _ in range(4))
o, lse = twfa.fa_fwd(fp, q, k, v, return_lse=True)
twfa.fa_bwd(bp, q, k, v, o, do, lse); torch.cuda.synchronize()
PY
TWFA_LIB=paper_2512_18134_b200/variants/bwdprof.so timeout 300 python /tmp/p.py 2>&1 | grep PROF | sort -k3 -n | head -60
