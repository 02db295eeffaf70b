"""Summarise an ncu --page source --print-source=sass CSV: hottest instructions by stall samples."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]; data = [r for r in rows[hi + 1:] if len(r) == len(h)]
si = h.index("Warp Stall Sampling (All Samples)"); ei = h.index("Instructions Executed")
tot = sum(float(r[si] or 0) for r in data)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
print("total samples", tot, "instructions", len(data))
for k, r in enumerate(data):
    r.append(k)
for r in sorted(data, key=lambda r: -float(r[si] or 0))[:n]:
    print(f"{r[-1]:5d} {100*float(r[si])/tot:5.1f}% exec={r[ei]:>10} {r[1][:100]}")
