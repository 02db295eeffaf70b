# compute-sanitizer on the final kernels: memcheck (smoke), racecheck and synccheck (small forward / backward)
mkdir -p gpurun_out/r02e
cat > /tmp/small.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import torch, paper_2512_18134_b200 as twfa
fp = twfa.Plan(*twfa.load_schedule("fa_fwd")); bp = twfa.Plan(*twfa.load_schedule("fa_bwd"))
for causal in (False, True):
    q, k, v, do = (torch.randn(1, 2, 384, 128, device="cuda").to(torch.bfloat16) for _ in range(4))
    o, lse = twfa.fa_fwd(fp, q, k, v, causal=causal, return_lse=True)
    twfa.fa_bwd(bp, q, k, v, o, do, lse, causal=causal)
torch.cuda.synchronize(); print("small ok")
PY
timeout 900 compute-sanitizer --tool memcheck python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02e/sanitizer_memcheck.txt 2>&1; tail -2 gpurun_out/r02e/sanitizer_memcheck.txt
timeout 900 compute-sanitizer --tool racecheck python /tmp/small.py > gpurun_out/r02e/sanitizer_racecheck.txt 2>&1; tail -3 gpurun_out/r02e/sanitizer_racecheck.txt
timeout 900 compute-sanitizer --tool synccheck python /tmp/small.py > gpurun_out/r02e/sanitizer_synccheck.txt 2>&1; tail -3 gpurun_out/r02e/sanitizer_synccheck.txt
