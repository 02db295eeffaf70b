# forward synccheck (every o_done phase awaited now), parity, and timing against the previous form
mkdir -p gpurun_out/r02e
cat > /tmp/fwd_only.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import torch, paper_2512_18134_b200 as twfa
fp = twfa.Plan(*twfa.load_schedule("fa_fwd"))
for pair in ("1", "0"):
    os.environ["TWFA_PAIR"] = pair
    for causal in (False, True):
        q, k, v = (torch.randn(1, 2, 640, 128, device="cuda").to(torch.bfloat16) for _ in range(3))
        twfa.fa_fwd(fp, q, k, v, causal=causal, return_lse=True)
torch.cuda.synchronize(); print("fwd only ok")
PY
timeout 900 compute-sanitizer --tool synccheck python /tmp/fwd_only.py > gpurun_out/r02e/sanitizer_synccheck_fwd.txt 2>&1; grep -c "Missing wait" gpurun_out/r02e/sanitizer_synccheck_fwd.txt; tail -2 gpurun_out/r02e/sanitizer_synccheck_fwd.txt
grep -A9 "Barrier error" gpurun_out/r02e/sanitizer_synccheck_fwd.txt | grep "Device Frame" | grep -o "fa_fwd_kernel.cuh:[0-9]*" | sort | uniq -c | head
timeout 600 python -m pytest tests/test_gpu_fa.py -x -q 2>&1 | tail -1
REPS=2 timeout 600 python tools/sustained.py paper_2512_18134_b200/libtwfa.so paper_2512_18134_b200/variants/crwait0.so
