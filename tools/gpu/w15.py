import sys, os, json, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2512_18134_b200 as twfa
prob, sol = twfa.load_schedule("fa_fwd")
plan = twfa.Plan(prob, sol)
ids = [n["id"] for n in json.loads(prob)["graph"]["nodes"]]
nw, cap = 16, 8192
tr = torch.zeros(nw * cap * 8, dtype=torch.int32, device="cuda")
q, k, v = (torch.randn(4, 32, 8192, 128, device="cuda").to(torch.bfloat16) for _ in range(3))
twfa.fa_fwd(plan, q, k, v); twfa.fa_fwd(plan, q, k, v, trace=tr, trace_cap=cap); torch.cuda.synchronize()
t = tr.cpu().numpy().view(np.uint32).reshape(nw, cap, 8).astype(np.int64)
w = 15
recs = [tuple(int(x) for x in t[w, 1 + i, :6]) for i in range(int(t[w, 0, 0]))]
t0 = min(r[3] for r in recs if r[2] == 30)
for r in recs:
    if r[2] in (30, 31):
        rd = (r[4] - t0) if r[4] else -1
        print(f"{ids[r[0]]:4s} it={r[1]:3d} trip={r[2]} issue={r[3]-t0:6d} ready={rd:6d} done={r[5]-t0:6d}")
