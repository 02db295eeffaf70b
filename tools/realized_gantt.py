#!/usr/bin/env python3
"""Realized schedule vs solved schedule.

One traced launch of the production kernel gives, on CTA 0, every op
instance each warp issued: (node, iteration, trip, issue, ready, done)
clocks. From it:

1. Rebuild the realized (M', A'). Stage = trip - iteration, slot from the
   solution; streamed loads use their due stage. Check (M', A') equals the
   solution, then pass it back through the unmodified reference validator
   (validate_program, sim.cpp:79-311, via oracle/_ref).
2. Render the solver's schedule with the reference's own Gantt
   (emit_gantt, viz.cpp:59-146).
3. Render the measured timeline of two steady trips: one row per warp, one
   box per op from inputs-ready to done, in SM clocks. Write it next to (2)
   under profiles/.

usage (GPU box): python tools/realized_gantt.py [schedule] [out_prefix]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))

COLORS = {"LD": "#4caf50", "S": "#e91e63", "PV": "#ad1457", "MX": "#2196f3", "EX": "#0d47a1", "CR": "#ffb300"}


def svg_timeline(recs, ids, warps, t0, t1, title):
    W, rowh, left = 1400, 22, 70
    scale = (W - left - 10) / max(1, t1 - t0)
    rows = sorted(warps)
    h = 40 + rowh * len(rows) + 20
    out = [f'<svg xmlns="http://www.w3.org/2000/svg" width="{W}" height="{h}" font-family="monospace" font-size="11">',
           f'<text x="5" y="15">{title}</text>']
    for i, w in enumerate(rows):
        y = 30 + i * rowh
        out.append(f'<text x="5" y="{y + 14}">warp {w}</text>')
        out.append(f'<line x1="{left}" y1="{y + rowh - 2}" x2="{W - 10}" y2="{y + rowh - 2}" stroke="#ddd"/>')
    for (w, node, it, trip, t_issue, t_ready, t_done) in recs:
        a, b = (t_ready or t_issue), t_done
        if b < t0 or a > t1:
            continue
        op = ids[node]
        kind = op.rstrip("0123456789")
        kind = "LD" if kind.startswith("LD") else kind
        x = left + (max(a, t0) - t0) * scale
        wd = max(1.0, (min(b, t1) - max(a, t0)) * scale)
        y = 30 + rows.index(w) * rowh
        out.append(f'<rect x="{x:.1f}" y="{y}" width="{wd:.1f}" height="{rowh - 6}" fill="{COLORS.get(kind, "#999")}">'
                   f'<title>{op} it={it} trip={trip} ready={a - t0} done={b - t0}</title></rect>')
        if wd > 28:
            out.append(f'<text x="{x + 2:.1f}" y="{y + 12}" fill="white">{op}</text>')
    out.append(f'<text x="{left}" y="{h - 5}">0 clk</text><text x="{W - 90}" y="{h - 5}">{t1 - t0} clk</text></svg>')
    return "\n".join(out)


def main():
    import numpy as np
    import torch
    import _weftsched as ws  # the unmodified reference (oracle/_ref)
    import paper_2512_18134_b200 as twfa
    name = sys.argv[1] if len(sys.argv) > 1 else "fa_fwd"
    prefix = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out", "realized_" + name)
    prob, sol = twfa.load_schedule(name)
    plan = twfa.Plan(prob, sol)
    desc = plan.describe()
    solution = json.loads(sol)
    ids = [n["id"] for n in json.loads(prob)["graph"]["nodes"]]
    nw, cap = desc["num_warps"], 8192
    tr = torch.zeros(nw * cap * 8, dtype=torch.int32, device="cuda")
    q, k, v = (torch.randn(4, 32, 8192, 128, device="cuda").to(torch.bfloat16) for _ in range(3))
    twfa.fa_fwd(plan, q, k, v)
    twfa.fa_fwd(plan, q, k, v, trace=tr, trace_cap=cap)
    torch.cuda.synchronize()
    t = tr.cpu().numpy().view(np.uint32).reshape(nw, cap, 8).astype(np.int64)
    recs = []
    for w in range(nw):
        for i in range(int(t[w, 0, 0])):
            e = t[w, 1 + i]
            trip = int(e[2]) - (1 << 32) if int(e[2]) >= 1 << 31 else int(e[2])  # trip -1 primes rings
            recs.append((w, int(e[0]), int(e[1]), trip, int(e[3]), int(e[4]), int(e[5])))
    I = solution["I"]
    prefetch = desc.get("prefetch", {})
    stage, warps = {}, {}
    for (w, node, it, trip, *_c) in recs:
        stage.setdefault(ids[node], set()).add(trip - it)
        warps.setdefault(ids[node], set()).add(w)
    m_real = {v: (solution["M"][v] // I if v in prefetch else min(stage[v])) * I + solution["M"][v] % I for v in ids}
    a_real = {v: min(warps[v]) for v in ids}
    realized = dict(solution, M=m_real, A=a_real)
    violations = ws.validate(prob, json.dumps(realized))
    report = {"schedule": name, "I": I, "realized_equals_solution": m_real == solution["M"] and a_real == solution["A"],
              "validate_program": violations,
              "streamed_loads_stage_range": {v: sorted(stage[v]) for v in prefetch}}
    # measured timeline: two steady trips of the first work tile
    mid = 30
    t0 = min(r[4] for r in recs if r[3] == mid)
    t_end = min(r[4] for r in recs if r[3] == mid + 2)
    steady = [r for r in recs if r[3] in (mid, mid + 1)]
    span = (t_end - t0) % (1 << 32)
    report["measured_clk_two_trips"] = span
    report["predicted_clk_two_trips"] = 2 * I * 256
    os.makedirs(os.path.dirname(prefix), exist_ok=True)
    with open(prefix + "_measured.svg", "w") as f:
        f.write(svg_timeline(steady, ids, {r[0] for r in steady}, t0, t0 + span,
                             f"{name}: measured, CTA 0, trips {mid}-{mid + 1} of work tile 0 "
                             f"({span} clk; solver predicts {2 * I * 256})"))
    with open(prefix + "_solved.svg", "w") as f:
        f.write(ws.gantt(prob, sol))
    with open(prefix + "_report.json", "w") as f:
        json.dump(report, f, indent=1)
    print(json.dumps(report, indent=1))


if __name__ == "__main__":
    main()
