"""Per-op wait / work statistics and one steady-state timeline of the FA
backward on CTA 0 (C3 shape, full grid), from the kernel's issue trace.
usage: python tools/bwd_trace_stats.py [schedule] [B H S]"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2512_18134_b200 as twfa
name = sys.argv[1] if len(sys.argv) > 1 else "fa_bwd"
B, H, S = (int(x) for x in sys.argv[2:5]) if len(sys.argv) > 4 else (4, 32, 8192)
prob, sol = twfa.load_schedule(name)
bplan = twfa.Plan(prob, sol)
fplan = twfa.Plan(*twfa.load_schedule("fa_fwd"))
ids = [n["id"] for n in json.loads(prob)["graph"]["nodes"]]
nw, cap = bplan.describe()["num_warps"], 4096
tr = torch.zeros(nw * cap * 8, dtype=torch.int32, device="cuda")
q, k, v, do = (torch.randn(B, H, S, 128, device="cuda").to(torch.bfloat16) for _ in range(4))
o, lse = twfa.fa_fwd(fplan, q, k, v, return_lse=True)
ws = None
for _ in range(2): twfa.fa_bwd(bplan, q, k, v, o, do, lse)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record(); twfa.fa_bwd(bplan, q, k, v, o, do, lse); e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
e0.record(); twfa.fa_bwd(bplan, q, k, v, o, do, lse, trace=tr, trace_cap=cap); e1.record(); torch.cuda.synchronize()
print(f"{name} B={B} H={H} S={S}: plain {ms:.3f} ms ({10 * B * H * S * S * 128 / ms / 1e9:.0f} TF/s), traced {e0.elapsed_time(e1):.3f} ms")
t = tr.cpu().numpy().view(np.uint32).reshape(nw, cap, 8).astype(np.int64)
recs = []
for w in range(nw):
    for i in range(int(t[w, 0, 0])):
        e = t[w, 1 + i]
        trip = int(e[2]) - (1 << 32) if int(e[2]) >= 1 << 31 else int(e[2])
        recs.append((w, ids[e[0]], int(e[1]), trip, int(e[3]), int(e[4]), int(e[5]), int(e[6])))
d = lambda a, b: (b - a) % (1 << 32)
print(f"{'op':4s} {'warp':>4s} {'n':>6s} {'ready_med':>9s} {'done_med':>9s} {'issue2issue':>11s}")
for op in ids:
    ws_ = sorted({r[0] for r in recs if r[1] == op})
    for w in ws_[:1]:
        rs = [r for r in recs if r[1] == op and r[0] == w and r[7] == 0]
        if len(rs) < 8: continue
        rd = np.array([d(r[4], r[5]) if r[5] else 0 for r in rs]); dn = np.array([d(r[4], r[6]) for r in rs])
        iss = np.array([d(a[4], b[4]) for a, b in zip(rs, rs[1:])])
        print(f"{op:4s} {w:4d} {len(rs):6d} {np.median(rd):9.0f} {np.median(dn):9.0f} {np.median(iss):11.0f}")
mid = 30
sel = [r for r in recs if r[7] == 0 and r[2] in (mid, mid + 1) and (r[0] % 4 == 0 or r[0] >= 12)]
t0 = min(r[4] for r in sel)
print(f"\niterations {mid}, {mid + 1} of work item 0 (CTA 0): warp op it trip issue ready done (clk from first)")
for r in sorted(sel, key=lambda r: r[4]):
    print(f"w{r[0]:2d} {r[1]:4s} it={r[2]:3d} trip={r[3]:3d} issue={d(t0, r[4]):6d} ready={d(t0, r[5]) if r[5] else -1:6d} done={d(t0, r[6]):6d}")
