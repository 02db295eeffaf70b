"""Which part of the forward trip grows in SM cycles with the SM clock?
Traced C3 launch (CTA 0) at the burst clock (idle GPU, ~1965 MHz) and again
after 3 s of back-to-back launches (power-capped, ~1600 MHz): per-op median
wait (issue -> inputs ready) and work (ready -> done) in clk, the trip, and
the effective clock (CTA 0's clock64 span over the launch time)."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2512_18134_b200 as twfa
prob, sol = twfa.load_schedule("fa_fwd")
plan = twfa.Plan(prob, sol)
ids = [n["id"] for n in json.loads(prob)["graph"]["nodes"]]
nw, cap = 16, 8192
tr = torch.zeros(nw * cap * 8, dtype=torch.int32, device="cuda")
q, k, v = (torch.randn(4, 32, 8192, 128, device="cuda").to(torch.bfloat16) for _ in range(3))
d = lambda a, b: (b - a) % (1 << 32)

def traced(tag):
    tr.zero_()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); twfa.fa_fwd(plan, q, k, v, trace=tr, trace_cap=cap); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    t = tr.cpu().numpy().view(np.uint32).reshape(nw, cap, 8).astype(np.int64)
    recs = [(w, ids[t[w, 1 + i, 0]], t[w, 1 + i]) for w in range(nw) for i in range(int(t[w, 0, 0]))]
    ts = np.array([r[2][3] for r in recs])
    span = d(ts.min(), ts.max())
    out = {"tag": tag, "launch_ms": round(ms, 3), "eff_mhz": round(span / (ms * 1e3))}
    for op in ("S1", "PV0", "S0", "PV1", "LDK", "LDV", "MX0", "MX1", "CR0"):
        ws = sorted({r[0] for r in recs if r[1] == op})
        rs = [r[2] for r in recs if r[1] == op and r[0] == ws[0]]
        rs = rs[len(rs) // 5:]
        wait = np.median([d(e[3], e[4]) for e in rs if e[4]]) if any(e[4] for e in rs) else 0
        work = np.median([d(e[4] or e[3], e[5]) for e in rs])
        out[op] = (int(wait), int(work))
    s1 = [r[2][3] for r in recs if r[1] == "S1" and r[0] == 15]
    out["trip"] = int(np.median(np.diff(s1) % (1 << 32)))
    print(json.dumps(out), flush=True)

for _ in range(3): twfa.fa_fwd(plan, q, k, v)
torch.cuda.synchronize()
traced("burst")
t0 = time.time()
while time.time() - t0 < 3.0:
    for _ in range(10): twfa.fa_fwd(plan, q, k, v)
    torch.cuda.synchronize()
traced("sustained")
