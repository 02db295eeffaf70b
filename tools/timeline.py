"""Per-warp timeline of the realized FA schedule (CTA 0) from the kernel trace."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2512_18134_b200 as twfa
S = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
prob, sol = twfa.load_schedule(sys.argv[2] if len(sys.argv) > 2 else "fa_fwd")
plan = twfa.Plan(prob, sol)
ids = [n["id"] for n in json.loads(prob)["graph"]["nodes"]]
nw, cap = 16, 2048
tr = torch.zeros(nw * cap * 8, dtype=torch.int32, device="cuda")
q, k, v = (torch.randn(1, 1, S, 128, device="cuda").to(torch.bfloat16) for _ in range(3))
twfa.fa_fwd(plan, q, k, v)  # warm
twfa.fa_fwd(plan, q, k, v, trace=tr, trace_cap=cap)
torch.cuda.synchronize()
t = tr.cpu().numpy().view(np.uint32).reshape(nw, cap, 8)
recs = []
for w in range(nw):
    for i in range(int(t[w, 0, 0])):
        e = t[w, 1 + i]
        recs.append((w, ids[e[0]], int(e[1]), int(e[2]), int(e[3]), int(e[4]), int(e[5])))
t0 = min(r[4] for r in recs)
N = S // 128
mid = N // 2
print("trip", mid, "and", mid + 1, "(times relative to trip start, cycles): warp op it issue ready done")
start = min(r[4] for r in recs if r[3] == mid)
for r in sorted(recs, key=lambda r: r[4]):
    if r[3] in (mid, mid + 1):
        rd = r[5] - start if r[5] else -1
        print(f"w{r[0]:2d} {r[1]:4s} it={r[2]:3d} trip={r[3]:3d} issue={r[4]-start:7d} ready={rd:7d} done={r[6]-start:7d} "
              f"wait={r[5]-r[4] if r[5] else 0:6d} work={r[6]-(r[5] or r[4]):6d}")
# per-op average wait / work over steady trips
print("\nsteady averages over trips 4..N-4:")
for op in ids:
    rs = [r for r in recs if r[1] == op and 4 <= r[3] < N - 4]
    if not rs: continue
    wait = np.mean([(r[5] - r[4]) if r[5] else 0 for r in rs]); work = np.mean([r[6] - (r[5] or r[4]) for r in rs])
    print(f"{op:4s} wait={wait:8.0f} work={work:8.0f} n={len(rs)}")
for op in ("S0", "S1", "PV0", "PV1", "LDK"):
    c = sorted(r[4] for r in recs if r[1] == op and r[0] == min(rr[0] for rr in recs if rr[1] == op))
    d = np.diff(c)
    print(op, "issue-to-issue median", np.median(d[4:-4]) if len(d) > 8 else d)
