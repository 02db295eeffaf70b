"""Rebuild the schedule a kernel actually ran from its issue trace and check
it against the solution JSON (test infrastructure for tests/test_gpu_trace.py).

A traced launch (twfa_fa_fwd_traced / twfa_fa_bwd_traced) records, for CTA 0,
every op instance each warp issued: (node, iteration, trip, clocks, work
tile ordinal, iterations of that tile). From it:

* A'(v): the warps v was issued from;
* stage'(v) = trip - iteration of every instance;
* the per-warp issue order, trip by trip, for every work tile the CTA ran
  (tiles of different lengths under causal work lists, several tiles per CTA
  with the next tile's loads and Q prefetched across the boundary).

The realized (M', A') -- stage' * I + (M mod I), min A' -- is what the
reference's validate_program (/root/reference/proj/src/sim.cpp:79-311) is run
on. Streamed loads (the reference's streaming rewrite, jointsolve.cpp:511-524:
zero-cycle, ring depth a free parameter) may issue up to `prefetch` trips
before their stage, never after it; a load of the next work tile issued while
the current one drains is the cross-tile form of the same latitude.
"""
import json

import numpy as np


def traced_records(trace, num_warps, cap):
    """[warp] -> list of (node, it, trip, t_issue, t_ready, t_done, tile, tile_n)."""
    t = trace.cpu().numpy().view(np.uint32).reshape(num_warps, cap, 8).astype(np.int64)
    out = {}
    for w in range(num_warps):
        n = int(t[w, 0, 0])
        recs = []
        for i in range(n):
            r = [int(x) for x in t[w, 1 + i]]
            r[2] = r[2] - (1 << 32) if r[2] >= 1 << 31 else r[2]  # trip -1 primes the rings
            recs.append(tuple(r))
        out[w] = recs
    return out


def check_realized(prob_json, sol_json, desc, per_warp, streamed=("LDK", "LDV", "LDQ", "LDO", "LDA", "LDB")):
    """Assert the trace realizes the solution; returns (M', A', tiles seen)."""
    prob, sol = json.loads(prob_json), json.loads(sol_json)
    nodes = prob["graph"]["nodes"]
    ids = [n["id"] for n in nodes]
    wreq = {n["id"]: n.get("warps_required", 1) for n in nodes}
    I = sol["I"]
    stage = {v: sol["M"][v] // I for v in ids}
    max_stage = max(stage.values())
    prefetch = desc.get("prefetch", {})
    loads = {v for v in ids if v in prefetch or v in streamed}
    realized_warps = {v: set() for v in ids}
    realized_stage = {v: set() for v in ids}
    tiles_seen = set()
    for w, recs in per_warp.items():
        if not recs:
            continue
        ops = [v for v in ids if sol["A"][v] <= w < sol["A"][v] + wreq[v]]
        ops.sort(key=lambda v: (sol["M"][v] % I, ids.index(v)))
        timed = [v for v in ops if v not in loads]
        # group this warp's records by work tile, in issue order
        first_timed = {}
        for k, r in enumerate(recs):
            if ids[r[0]] not in loads:
                first_timed.setdefault(r[6], k)
        tiles = []
        for r in recs:
            if r[6] not in tiles:
                tiles.append(r[6])
        for tile in tiles:
            tiles_seen.add(tile)
            trs = [r for r in recs if r[6] == tile]
            N = trs[0][7]
            assert all(r[7] == N for r in trs), f"warp {w} tile {tile}: inconsistent iteration counts"
            expect = [(ids.index(v), it, r) for r in range(N + max_stage) for v in timed
                      for it in [r - stage[v]] if 0 <= it < N]
            got = [r[:3] for r in trs if ids[r[0]] not in loads]
            assert got == expect, f"warp {w} tile {tile}: issue order differs from the trip program"
            for v in [v for v in ops if v in loads]:
                lrs = [(k, r) for k, r in enumerate(recs) if r[6] == tile and ids[r[0]] == v]
                assert [r[1] for _, r in lrs] == list(range(N)), f"{v} tile {tile}: iterations out of order"
                for k, r in lrs:
                    if k < first_timed.get(tile, len(recs)):
                        continue  # issued while the previous tile drained (cross-tile prefetch)
                    realized_stage[v].add(r[2] - r[1])
            for r in trs:
                realized_warps[ids[r[0]]].add(w)
                if ids[r[0]] not in loads:
                    realized_stage[ids[r[0]]].add(r[2] - r[1])
    for v in ids:
        a = sol["A"][v]
        assert realized_warps[v] == set(range(a, a + wreq[v])), (v, realized_warps[v])
        if v in loads:
            pf = prefetch.get(v, 1)
            assert realized_stage[v] <= set(range(stage[v] - pf, stage[v] + 1)), (v, realized_stage[v])
        else:
            assert realized_stage[v] == {stage[v]}, (v, realized_stage[v])
    m_real = {v: (stage[v] if v in loads else min(realized_stage[v])) * I + sol["M"][v] % I for v in ids}
    a_real = {v: min(realized_warps[v]) for v in ids}
    return m_real, a_real, tiles_seen
