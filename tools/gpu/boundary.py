import sys, os, json, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2512_18134_b200 as twfa
prob, sol = twfa.load_schedule("fa_fwd")
plan = twfa.Plan(prob, sol)
ids = [n["id"] for n in json.loads(prob)["graph"]["nodes"]]
nw, cap = 16, 8192
tr = torch.zeros(nw * cap * 8, dtype=torch.int32, device="cuda")
S = int(os.environ.get("S", "8192"))
q, k, v = (torch.randn(4, 32, S, 128, device="cuda").to(torch.bfloat16) for _ in range(3))
twfa.fa_fwd(plan, q, k, v); twfa.fa_fwd(plan, q, k, v, trace=tr, trace_cap=cap); torch.cuda.synchronize()
t = tr.cpu().numpy().view(np.uint32).reshape(nw, cap, 8).astype(np.int64)
recs = []
for w in (0, 3, 4, 7, 8, 11, 15):
    for i in range(int(t[w, 0, 0])):
        e = [int(x) for x in t[w, 1 + i, :6]]
        if e[2] >= 1 << 31: e[2] -= 1 << 32
        recs.append((w, *e))
# first boundary: records of work tile 0 trips >= 62 and work tile 1 trips <= 2 (by time order on warp 15)
w15 = [r for r in recs if r[0] == 15]
# find index where iteration resets
idx = next(i for i in range(1, len(w15)) if w15[i][3] < w15[i - 1][3] - 5)
tb = w15[idx][4]
t0 = tb - 12000
for r in sorted(recs, key=lambda r: r[4]):
    if t0 <= r[4] <= tb + 12000:
        print(f"w{r[0]:2d} {ids[r[1]]:4s} it={r[2]:3d} trip={r[3]:3d} issue={r[4]-tb:7d} ready={(r[5]-tb) if r[5] else 0:7d} done={r[6]-tb:7d}")
