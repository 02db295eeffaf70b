"""Time the FA backward for each library given (TWFA_LIB per subprocess)."""
import os, subprocess, sys
code = r'''
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2512_18134_b200 as twfa
fp = twfa.Plan(*twfa.load_schedule("fa_fwd")); bp = twfa.Plan(*twfa.load_schedule(os.environ.get("BSCHED", "fa_bwd")))
B, H, S = [int(x) for x in os.environ.get("SHAPE", "4,32,8192").split(",")]
causal = os.environ.get("CAUSAL", "0") == "1"
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
print(f"{os.path.basename(os.environ['TWFA_LIB'])} bwd B={B} H={H} S={S} causal={causal}: {ms:.3f} ms {fl/ms/1e9:.1f} TFLOPS", flush=True)
'''
for lib in sys.argv[1:]:
    env = dict(os.environ, TWFA_LIB=os.path.abspath(lib))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    print(r.stdout.strip() or r.stderr[-1500:], flush=True)
