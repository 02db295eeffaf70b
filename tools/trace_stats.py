"""Per-op wait / work statistics of the realized FA schedule on CTA 0 under a
full-size launch (all SMs busy), from the kernel's issue trace.
usage: python tools/trace_stats.py B H S [schedule] [causal]"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2512_18134_b200 as twfa
B, H, S = (int(x) for x in sys.argv[1:4])
name = sys.argv[4] if len(sys.argv) > 4 else "fa_fwd"
causal = len(sys.argv) > 5 and sys.argv[5] == "1"
if ":" in name:  # problem:solution-path (experiments)
    pn, sp = name.split(":")
    prob = twfa.load_schedule(pn)[0]
    sol = open(os.path.join(twfa.schedule_dir(), sp + ".solution.json")).read()
else:
    prob, sol = twfa.load_schedule(name)
plan = twfa.Plan(prob, sol)
ids = [n["id"] for n in json.loads(prob)["graph"]["nodes"]]
nw, cap = plan.describe()["num_warps"], 8192
tr = torch.zeros(nw * cap * 8, dtype=torch.int32, device="cuda")
q, k, v = (torch.randn(B, H, S, 128, device="cuda").to(torch.bfloat16) for _ in range(3))
for _ in range(2): twfa.fa_fwd(plan, q, k, v, causal=causal)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); twfa.fa_fwd(plan, q, k, v, causal=causal); e1.record(); torch.cuda.synchronize()
ms_plain = e0.elapsed_time(e1)
e0.record(); twfa.fa_fwd(plan, q, k, v, causal=causal, trace=tr, trace_cap=cap); e1.record()
torch.cuda.synchronize()
print(f"{name} B={B} H={H} S={S}: plain {ms_plain:.3f} ms, traced {e0.elapsed_time(e1):.3f} ms")
t = tr.cpu().numpy().view(np.uint32).reshape(nw, cap, 8).astype(np.int64)
recs = []
for w in range(nw):
    for i in range(int(t[w, 0, 0])):
        e = t[w, 1 + i]
        trip = int(e[2]) - (1 << 32) if int(e[2]) >= 1 << 31 else int(e[2])  # trip -1 primes rings
        recs.append((w, ids[e[0]], int(e[1]), trip, int(e[3]), int(e[4]), int(e[5])))
def d(a, b):
    return (b - a) % (1 << 32)
print(f"{'op':4s} {'warp':>4s} {'n':>6s} {'wait_med':>9s} {'work_med':>9s} {'wait_mean':>9s} {'work_mean':>9s} {'issue2issue':>11s}")
for op in ids:
    for w in sorted({r[0] for r in recs if r[1] == op}):
        rs = [r for r in recs if r[1] == op and r[0] == w]
        if len(rs) < 8: continue
        wait = np.array([d(r[4], r[5]) if r[5] else 0 for r in rs]); work = np.array([d(r[5] or r[4], r[6]) for r in rs])
        iss = np.array([d(a[4], b[4]) for a, b in zip(rs, rs[1:])])
        print(f"{op:4s} {w:4d} {len(rs):6d} {np.median(wait):9.0f} {np.median(work):9.0f} {wait.mean():9.0f} {work.mean():9.0f} {np.median(iss):11.0f}")
        if w != min(r[0] for r in recs if r[1] == op): continue
# one steady trip, all warps, relative times
mid = 30
start = min(r[4] for r in recs if r[3] == mid)
print(f"\ntrip {mid}..{mid+1} of work tile 0: warp op it issue ready done")
for r in sorted(recs, key=lambda r: r[4]):
    if r[3] in (mid, mid + 1) and d(start, r[4]) < 20000 and (r[0] % 4 == 0 or r[0] >= 12 or r[1][0] in "SP"):
        print(f"w{r[0]:2d} {r[1]:4s} it={r[2]:3d} trip={r[3]:3d} issue={d(start, r[4]):6d} ready={d(start, r[5]) if r[5] else -1:6d} done={d(start, r[6]):6d}")

# tile boundaries: time from the last steady issue of each op to its first
# issue in the next work tile, in units of the median trip
print("\nwork-tile boundary cost (CTA 0), per op: median gap across a tile boundary / median trip")
for op in ids:
    for w in sorted({r[0] for r in recs if r[1] == op})[:1]:
        rs = [r for r in recs if r[1] == op and r[0] == w]
        if len(rs) < 8: continue
        steady, bound = [], []
        for a, b in zip(rs, rs[1:]):
            (bound if b[2] < a[2] else steady).append(d(a[4], b[4]))
        if steady and bound:
            print(f"{op:4s} w{w:2d} trip {np.median(steady):7.0f}  boundary {np.median(bound):8.0f} "
                  f"({np.median(bound) / np.median(steady):.2f} trips)  n={len(bound)}")
