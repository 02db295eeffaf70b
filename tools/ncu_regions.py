"""Per-role stall breakdown of an ncu source capture (--page source --csv
--print-source=sass): the SASS is split into regions at changes of the
per-instruction execution count class; prints the hot instructions and the
stall reasons of the region holding the tcgen05.mma issues (the MMA warp).
usage: python tools/ncu_regions.py <source.csv> [top_n]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]
data = [r for r in rows[hi + 1:] if len(r) == len(h)]
si = h.index("Warp Stall Sampling (All Samples)")
ei = h.index("Instructions Executed")
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
ri = [h.index(c) for c in reasons]
tot = sum(float(r[si] or 0) for r in data)
top = int(sys.argv[2]) if len(sys.argv) > 2 else 60
mma = [k for k, r in enumerate(data) if "UTCHMMA" in r[1] or "UTCQMMA" in r[1]]
print(f"total samples {tot:.0f}; {len(data)} instructions; UTCHMMA at {mma[:4]}..{mma[-4:]}")
lo, hi2 = max(0, mma[0] - 120), min(len(data), mma[-1] + 60)
reg = data[lo:hi2]
rs = sum(float(r[si] or 0) for r in reg)
agg = {c: sum(float(r[i] or 0) for r in reg) for c, i in zip(reasons, ri)}
print(f"MMA-warp window [{lo}, {hi2}): {rs:.0f} samples ({100 * rs / tot:.1f}% of all)")
print("  " + ", ".join(f"{c[6:]} {100 * v / max(rs, 1):.1f}%" for c, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
for k, r in enumerate(reg):
    s = float(r[si] or 0)
    if s < rs * 0.004 and "UTCHMMA" not in r[1] and "UTCBAR" not in r[1] and "UTMALDG" not in r[1]:
        continue
    why = sorted(((float(r[i] or 0), c[6:]) for c, i in zip(reasons, ri)), reverse=True)[:2]
    print(f"{lo + k:5d} {s:6.0f} exec={r[ei]:>9} {r[1].strip()[:70]:70s} {why}")
