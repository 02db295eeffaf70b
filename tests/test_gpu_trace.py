"""The realized schedule is the solver's schedule.

The FA kernel records, for CTA 0, every op instance each warp issues:
(node, iteration, trip, clock64). From that trace we rebuild the schedule the
hardware actually ran -- warp range A'(v), stage' = trip - iteration, and the
issue order inside a trip -- and require it to equal the solution JSON
bit-for-bit (I, M div I, M mod I order, A). The realized (M', A') is then fed
back through the unmodified reference validator (validate_program,
/root/reference/proj/src/sim.cpp:79-311, via the oracle/_ref pybind module)
which must report no violations. Steady-state cycles per trip are measured
from the clock stamps and reported against I x (raw cycles per unit).
"""
import json
import os
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ref():
    sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))
    try:
        import _weftsched
    except ImportError:
        pytest.skip("oracle/_ref not built")
    return _weftsched


def realized_schedule(twfa, plan, B=1, H=1, S=2048, causal=False, cap=512):
    desc = plan.describe()
    nw = desc["num_warps"]
    trace = torch.zeros(nw * cap * 8, dtype=torch.int32, device="cuda")
    dev = torch.device("cuda:0")
    q, k, v = (torch.randn(B, H, S, 128, device=dev).to(torch.bfloat16) for _ in range(3))
    twfa.fa_fwd(plan, q, k, v, causal=causal, trace=trace, trace_cap=cap)
    torch.cuda.synchronize()
    t = trace.cpu().numpy().view(np.uint32).reshape(nw, cap, 8)
    per_warp = {}
    for w in range(nw):
        n = int(t[w, 0, 0])
        # (node, iteration, trip, t_issue, t_ready, t_done)
        # trip is signed: streamed loads prime their ring in trip -1
        per_warp[w] = [tuple(int(x) for x in t[w, 1 + i, :6]) for i in range(n)]
        per_warp[w] = [(r[0], r[1], r[2] - (1 << 32) if r[2] >= 1 << 31 else r[2]) + r[3:] for r in per_warp[w]]
    return desc, per_warp


def test_realized_schedule_is_the_solution(twfa):
    prob, sol = twfa.load_schedule("fa_fwd")
    plan = twfa.Plan(prob, sol)
    desc, per_warp = realized_schedule(twfa, plan)
    solution = json.loads(sol)
    names = list(json.loads(prob)["graph"]["nodes"])
    ids = [n["id"] for n in names]
    I = solution["I"]
    N = 2048 // 128
    realized_warps = {v: set() for v in ids}
    realized_stage = {v: set() for v in ids}
    for w, recs in per_warp.items():
        for node, it, trip, *_clk in recs:
            realized_warps[ids[node]].add(w)
            realized_stage[ids[node]].add(trip - it)
    # Streamed loads (variable latency, no predecessors: the reference's
    # streaming rewrite, jointsolve.cpp:511-524, turns them into zero-cycle ops
    # whose ring depth is a free parameter) fill a ring of depth D: the load of
    # iteration i may issue up to `prefetch` trips before the trip its
    # stage names, never after it. Every other op issues exactly in its stage.
    prefetch = desc.get("prefetch", {})
    for v in ids:
        a = solution["A"][v]
        wr = next(n.get("warps_required", 1) for n in names if n["id"] == v)
        assert realized_warps[v] == set(range(a, a + wr)), (v, realized_warps[v])
        st = solution["M"][v] // I
        if v in prefetch:
            assert realized_stage[v] <= set(range(st - prefetch[v], st + 1)), (v, realized_stage[v])
        else:
            assert realized_stage[v] == {st}, (v, realized_stage[v])
    # issue order inside each trip on each warp: by M mod I, then declaration order
    for w, recs in per_warp.items():
        expect = []
        ops = [v for v in ids if solution["A"][v] <= w < solution["A"][v]
               + next(n.get("warps_required", 1) for n in names if n["id"] == v)]
        ops.sort(key=lambda v: (solution["M"][v] % I, ids.index(v)))
        max_stage = max(solution["M"][v] // I for v in ids)
        # streamed loads: each iteration exactly once, in iteration order
        for v in [v for v in ops if v in prefetch]:
            its = [rec[1] for rec in recs if rec[0] == ids.index(v)]
            assert its == list(range(N)), f"{v} iterations {its}"
        # every other op of the warp: exactly the trip program, trip by trip
        timed = [v for v in ops if v not in prefetch]
        for r in range(N + max_stage):
            for v in timed:
                it = r - solution["M"][v] // I
                if 0 <= it < N:
                    expect.append((ids.index(v), it, r))
        got = [rec[:3] for rec in recs if ids[rec[0]] not in prefetch]
        assert got == expect, f"warp {w} issue order differs"

    # realized (M', A') back through the reference validator
    m_real = {v: (solution["M"][v] // I if v in prefetch else min(realized_stage[v])) * I + solution["M"][v] % I
              for v in ids}
    a_real = {v: min(realized_warps[v]) for v in ids}
    realized = dict(solution, M=m_real, A=a_real)
    ws = _ref()
    assert ws.validate(prob, json.dumps(realized)) == []
    assert m_real == solution["M"] and a_real == solution["A"]


def test_steady_state_cycles_per_trip(twfa):
    prob, sol = twfa.load_schedule("fa_fwd")
    plan = twfa.Plan(prob, sol)
    desc, per_warp = realized_schedule(twfa, plan, S=8192, cap=1024)
    meta = json.load(open(os.path.join(twfa.schedule_dir(), "fa_fwd.meta.json")))
    unit = 256  # raw B200 cycles per normalized unit (tools/make_problems.py)
    predicted = desc["I"] * unit
    # the MMA warp issuing S1: clock of consecutive steady-state issues
    s1 = [i for i, n in enumerate(json.loads(prob)["graph"]["nodes"]) if n["id"] == "S1"][0]
    w = json.loads(sol)["A"]["S1"]
    clk = np.array([rec[3] for rec in per_warp[w] if rec[0] == s1], dtype=np.int64)
    d = np.diff(clk) % (1 << 32)
    steady = float(np.median(d[4:-4])) if len(d) > 8 else float(np.median(d))
    print(f"\nsteady-state cycles per trip: measured {steady:.0f}, predicted I*unit = {predicted} "
          f"(F = {meta['F']})")
    assert steady > 0
