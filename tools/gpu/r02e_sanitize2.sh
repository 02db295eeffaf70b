# synccheck / racecheck on the backward alone (O and LSE from a torch fp32 forward)
mkdir -p gpurun_out/r02e
cat > /tmp/bwd_only.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import torch, paper_2512_18134_b200 as twfa
bp = twfa.Plan(*twfa.load_schedule("fa_bwd"))
for causal in (False, True):
    q, k, v, do = (torch.randn(1, 2, 384, 128, device="cuda").to(torch.bfloat16) for _ in range(4))
    s = (q.float() @ k.float().transpose(-1, -2)) / 128 ** 0.5
    if causal:
        s = s.masked_fill(torch.ones(384, 384, device="cuda", dtype=torch.bool).triu(1), float("-inf"))
    lse = torch.logsumexp(s, -1)
    o = (torch.softmax(s, -1) @ v.float()).to(torch.bfloat16)
    twfa.fa_bwd(bp, q, k, v, o, do, lse.contiguous(), causal=causal)
torch.cuda.synchronize(); print("bwd only ok")
PY
timeout 900 compute-sanitizer --tool synccheck python /tmp/bwd_only.py > gpurun_out/r02e/sanitizer_synccheck_bwd.txt 2>&1; tail -3 gpurun_out/r02e/sanitizer_synccheck_bwd.txt
timeout 900 compute-sanitizer --tool memcheck python /tmp/bwd_only.py > gpurun_out/r02e/sanitizer_memcheck_bwd.txt 2>&1; tail -2 gpurun_out/r02e/sanitizer_memcheck_bwd.txt
