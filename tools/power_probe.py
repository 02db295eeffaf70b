"""SM clock, power draw and throttle reasons sampled (NVML, every 20 ms) while a
kernel runs back to back for ~3 s: ours (C3 forward, pair and single CTA) and
cuDNN SDPA on the same shape. Also the in-kernel clock: CTA 0's traced
clock64 span over the launch time (effective SM MHz during the kernel)."""
import os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, pynvml
import torch.nn.functional as F
import paper_2512_18134_b200 as twfa
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
B, H, S = 4, 32, 8192
q, k, v = (torch.randn(B, H, S, 128, device="cuda").to(torch.bfloat16) for _ in range(3))
plan = twfa.Plan(*twfa.load_schedule("fa_fwd"))
fl = 4 * B * H * S * S * 128

def sample(stop, out):
    while not stop.is_set():
        out.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                    pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                    pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)))
        time.sleep(0.02)

def run(name, fn, secs=3.0):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    stop, out = threading.Event(), []
    th = threading.Thread(target=sample, args=(stop, out)); th.start()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    n = 0; t0 = time.time(); e0.record()
    while time.time() - t0 < secs:
        for _ in range(20): fn()
        n += 20
        torch.cuda.synchronize()
    e1.record(); torch.cuda.synchronize()
    stop.set(); th.join()
    ms = e0.elapsed_time(e1) / n
    a = np.array([(c, p) for c, p, _ in out[len(out) // 5:]])
    reasons = 0
    for _, _, r in out: reasons |= r
    print(f"{name}: {ms:.3f} ms {fl / ms / 1e9:.0f} TF/s  sm_mhz median {np.median(a[:, 0]):.0f} "
          f"(min {a[:, 0].min():.0f})  power median {np.median(a[:, 1]):.0f} W  reasons 0x{reasons:x}", flush=True)

for pair in ("1", "0"):
    os.environ["TWFA_PAIR"] = pair
    run(f"twfa pair={pair}", lambda: twfa.fa_fwd(plan, q, k, v))
    # in-kernel clock of CTA 0 over the traced launch
    cap = 8192
    tr = torch.zeros(16 * cap * 8, dtype=torch.int32, device="cuda")
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); twfa.fa_fwd(plan, q, k, v, trace=tr, trace_cap=cap); e1.record(); torch.cuda.synchronize()
    t = tr.cpu().numpy().view(np.uint32).reshape(16, cap, 8).astype(np.int64)
    ts = [t[w, 1:1 + int(t[w, 0, 0]), 3] for w in range(16) if t[w, 0, 0] > 0]
    ts = np.concatenate(ts)
    span = (ts.max() - ts.min()) % (1 << 32)
    print(f"  traced launch {e0.elapsed_time(e1):.3f} ms, CTA 0 clock64 span {span} clk -> "
          f"{span / (e0.elapsed_time(e1) * 1e3):.0f} MHz effective", flush=True)
run("cudnn sdpa", lambda: F.scaled_dot_product_attention(q, k, v))
