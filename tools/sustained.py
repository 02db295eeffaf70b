"""Per-clock efficiency of kernel variants under sustained (power-capped) load.

Each variant (library path, optional ENV=VAL settings joined with '+', e.g.
`lib.so+TWFA_PAIR=0`) runs the C3 forward back to back for SECS seconds in its
own process while NVML samples the SM clock and power every 20 ms. Reported:
TF/s, median SM MHz under load, power, and the tensor-pipe fraction per clock
= TF/s / (SMs x 8192 flop/clk x MHz): the number a power cap cannot move.
usage: python tools/sustained.py VARIANT [VARIANT ...]   (SHAPE=B,H,S CAUSAL=1 SCHED=... REPS=n)"""
import os, subprocess, sys
code = r'''
import os, sys, threading, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch, pynvml
import paper_2512_18134_b200 as twfa
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
sched = os.environ.get("SCHED", "fa_fwd")
if ":" in sched:
    pn, sp = sched.split(":")
    plan = twfa.Plan(twfa.load_schedule(pn)[0], open(os.path.join(twfa.schedule_dir(), sp + ".solution.json")).read())
else:
    plan = twfa.Plan(*twfa.load_schedule(sched))
B, H, S = [int(x) for x in os.environ.get("SHAPE", "4,32,8192").split(",")]
causal = os.environ.get("CAUSAL", "0") == "1"
q, k, v = (torch.randn(B, H, S, 128, device="cuda").to(torch.bfloat16) for _ in range(3))
fl = 4 * B * H * S * S * 128 / (2 if causal else 1)
fn = lambda: twfa.fa_fwd(plan, q, k, v, causal=causal)
for _ in range(5): fn()
torch.cuda.synchronize()
samples, stop = [], threading.Event()
def smp():
    while not stop.is_set():
        samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), pynvml.nvmlDeviceGetPowerUsage(h) / 1e3))
        time.sleep(0.02)
th = threading.Thread(target=smp); th.start()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
secs = float(os.environ.get("SECS", "2.5")); n = 0; t0 = time.time(); e0.record()
while time.time() - t0 < secs:
    for _ in range(10): fn()
    n += 10; torch.cuda.synchronize()
e1.record(); torch.cuda.synchronize(); stop.set(); th.join()
ms = e0.elapsed_time(e1) / n
a = np.array(samples[len(samples) // 4:])
mhz = float(np.median(a[:, 0])); tf = fl / ms / 1e9
sms = torch.cuda.get_device_properties(0).multi_processor_count
print(f"{os.environ['VARIANT']:45s} {tf:7.1f} TF/s  {mhz:5.0f} MHz  {np.median(a[:, 1]):4.0f} W  "
      f"tensor/clk {tf * 1e12 / (sms * 8192 * mhz * 1e6):.3f}", flush=True)
'''
reps = int(os.environ.get("REPS", "1"))
for rep in range(reps):
    for var in sys.argv[1:]:
        lib, *envs = var.split("+")  # lib.so+ENV=VAL+ENV=VAL
        env = dict(os.environ, TWFA_LIB=os.path.abspath(lib), VARIANT=os.path.basename(var))
        for e in envs:
            kk, vv = e.split("=", 1)
            env[kk] = vv
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
        print(r.stdout.strip() or r.stderr[-1500:], flush=True)
