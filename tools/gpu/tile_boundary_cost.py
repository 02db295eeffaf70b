"""Cycles per K/V trip of CTA 0 (tile boundaries included) at C5 sequence lengths: the per-tile
boundary cost is the excess over the long-sequence trip time. trace_cap=2: only CTA 0's clock stamps."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2512_18134_b200 as twfa
plan = twfa.Plan(*twfa.load_schedule("fa_fwd"))
d = plan.describe()
sms = torch.cuda.get_device_properties(0).multi_processor_count
units, rows = sms // 2, 512
res = {}
for S in (1024, 2048, 4096, 8192):
    B, H = 16, 64 if S <= 2048 else 16
    q, k, v = (torch.randn(B, H, S, 128, device="cuda").to(torch.bfloat16) for _ in range(3))
    tr = torch.zeros(d["num_warps"] * 2 * 8, dtype=torch.int32, device="cuda")
    twfa.fa_fwd(plan, q, k, v)
    twfa.fa_fwd(plan, q, k, v, trace=tr, trace_cap=2)
    torch.cuda.synchronize()
    w = tr[:5].cpu().numpy().view(np.uint32).astype(np.int64)
    span = (w[3] - w[1]) % (1 << 32)
    tiles = B * H * (S // rows)
    my_tiles = -(-tiles // units)
    trips = my_tiles * (S // 128)
    res[S] = (span / trips, span / my_tiles, S // 128)
    print(f"S={S}: {my_tiles} tiles x {S // 128} trips on CTA 0, {span / trips:.0f} clk per trip, {span / my_tiles:.0f} per tile")
base = res[8192][0]
for S, (pt, ptile, n) in res.items():
    print(f"S={S}: boundary cost per tile ~ {ptile - n * base:.0f} clk (vs {base:.0f} clk per trip at S=8192)")
