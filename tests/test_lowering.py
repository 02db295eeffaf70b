"""The lowering (solution JSON -> per-warp trip programs) against the
reference's own consumer of the same documents.

The unmodified reference (weftsched, built in place into oracle/_ref) renders
a solution with `codegen` (synthesize, /root/reference/proj/src/codegen.cpp:
43-189). Its steady-state region lists every op once with its warp range, its
cycle inside the trip (M mod I) and the copy it belongs to (copy = copies - 1 -
stage). The executor's plan must carry exactly that: same I, same warp ranges,
same stages, and per warp the same op order as the reference's region order.
Document-level errors must be rejected like the reference rejects them
(solution_from_json, cli.cpp:96-155 -> ValueError in Python)."""
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ws():
    sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))
    try:
        import _weftsched
    except ImportError:
        pytest.skip("oracle/_ref not built")
    return _weftsched


def steady_programs_from_reference(ws, prob, sol):
    prog = json.loads(ws.codegen(prob, sol, "json"))
    copies = prog["copies"]
    per_warp, stage, warp = {}, {}, {}
    streamed = set(json.loads(sol).get("streaming_depths", {}))
    cycle = {}
    for ins in prog["steady_state"]:
        if ins["kind"] != "op":
            continue
        stage[ins["node"]] = copies - 1 - ins["copy"]
        warp[ins["node"]] = (ins["warp_start"], ins["warp_count"])
        cycle[ins["node"]] = ins["cycle"]
        for w in range(ins["warp_start"], ins["warp_start"] + ins["warp_count"]):
            per_warp.setdefault(w, []).append(ins["node"])
    # the executor issues streamed (zero-cycle) loads after the timed ops of
    # their cycle (lowering.cpp); otherwise the reference's region order
    for w, ops in per_warp.items():
        ops.sort(key=lambda v: (cycle[v], v in streamed))
    return prog, per_warp, stage, warp


@pytest.mark.parametrize("name", ["fa_fwd", "gemm_mainloop", "fa_bwd", "fa_bwd_pp"])
def test_plan_equals_reference_program(twfa, ws, name):
    prob, sol = twfa.load_schedule(name)
    d = twfa.Plan(prob, sol).describe()
    prog, per_warp, stage, warp = steady_programs_from_reference(ws, prob, sol)
    s = json.loads(sol)
    assert d["I"] == prog["I"] == s["I"]
    assert d["L"] == s["L"] and d["copies"] == prog["copies"]
    for v, nd in d["nodes"].items():
        assert nd["stage"] == stage[v] == s["M"][v] // s["I"]
        assert nd["slot"] == s["M"][v] % s["I"]
        assert (nd["warp_start"], nd["warp_count"]) == warp[v]
        assert nd["warp_start"] == s["A"][v]
    assert {int(w): p for w, p in d["warp_programs"].items()} == per_warp


def test_golden_solution_is_valid_under_the_reference(twfa, ws):
    for name in ("fa_fwd", "gemm_mainloop"):
        prob, sol = twfa.load_schedule(name)
        assert ws.validate(prob, sol) == []


def test_golden_problem_normalizes_to_committed(twfa, ws):
    """The committed normalized problem is the reference `normalize` of the raw
    B200 cost model (exact at U = 7, F = 0)."""
    d = twfa.schedule_dir()
    raw = open(os.path.join(d, "fa_fwd.raw.json")).read()
    meta = json.load(open(os.path.join(d, "fa_fwd.meta.json")))
    r = ws.normalize(raw, meta["resolution"])
    assert json.loads(r["problem"]) == json.loads(open(os.path.join(d, "fa_fwd.json")).read())
    assert r["F"] == 0


def test_gemm_stream_depth_sets_ring(twfa, ws):
    prob, _ = twfa.load_schedule("gemm_mainloop")
    for depth in (2, 3, 4):
        r = ws.joint(prob, 0, depth, "")
        d = twfa.Plan(prob, r["solution_json"]).describe()
        assert d["rings"]["AB"] == depth
        assert d["mma_warp"] == r["A"]["MMA"] and d["load_warp"] == r["A"]["LDA"]


def test_fa_ring_depth_follows_solution(twfa):
    prob, sol = twfa.load_schedule("fa_fwd")
    s = json.loads(sol)
    assert twfa.Plan(prob, sol).describe()["rings"] == {"K": 2, "V": 2, "S": 1}
    # one CTA per tile: two 32 KiB Q tiles + 2 + 2 ring slots of 32 KiB fill
    # the 227 KiB of shared memory. A deeper ring fits with the CTA-pair
    # realization (16 KiB K / V slots per CTA), which the plan then requires;
    # deeper than 4 is not realizable and must say so
    s["streaming_depths"] = {"LDK": 3, "LDV": 3}
    d = twfa.Plan(prob, json.dumps(s)).describe()
    assert d["rings"] == {"K": 3, "V": 3, "S": 1} and d["cta_pair"] is True
    s["streaming_depths"] = {"LDK": 5, "LDV": 2}
    with pytest.raises(ValueError, match="ring depth above 4"):
        twfa.Plan(prob, json.dumps(s))


@pytest.mark.parametrize("mutate,msg", [
    (lambda s: s.update(I=0), "positive integer I"),
    (lambda s: s.update(bogus=1), "unknown solution key"),
    (lambda s: s["M"].pop("S0"), "cover every node"),
    (lambda s: s["M"].update(S0=99), "does not fit in L"),
    (lambda s: s["A"].update(MX0=3), "warp_uniqueness.*aligned slot"),
    (lambda s: s["A"].update(EX0=8, MX0=4), "register_limit|share a warpgroup"),
    (lambda s: s["A"].update(S0=16), "warp_uniqueness.*aligned slot"),
    (lambda s: s.update(streaming_depths={"LDK": 1, "LDV": 1}), "shallower than its consumer lag|cannot run ahead"),
])
def test_bad_or_unrealizable_solutions_are_rejected(twfa, mutate, msg):
    prob, sol = twfa.load_schedule("fa_fwd")
    s = json.loads(sol)
    mutate(s)
    with pytest.raises(ValueError, match=msg):
        twfa.Plan(prob, json.dumps(s))


def test_reference_fixtures_without_a_b200_realization_are_rejected(twfa, ws):
    # the reference's own Fig. 1 attention problem (S, P, O on TC/MFU,
    # proj/tests/testutil.hpp:16-40) names ops the executor has no kernel for
    prob = json.dumps({
        "machine": {"units": [{"name": "TC", "capacity": 1}, {"name": "MFU", "capacity": 1}],
                    "memories": [{"name": "smem", "capacity": 1024}], "num_warps": 4, "reg_limit": 256,
                    "vl_warp": 3},
        "graph": {"nodes": [{"id": "S", "rrt": {"TC": [1]}, "cycles": 1},
                            {"id": "P", "rrt": {"MFU": [1]}, "cycles": 1},
                            {"id": "O", "rrt": {"TC": [1]}, "cycles": 1}],
                  "edges": [{"src": "S", "dst": "P", "d": 1}, {"src": "P", "dst": "O", "d": 1},
                            {"src": "O", "dst": "O", "d": 1, "delta": 1}]}})
    r = ws.joint(prob)
    assert (r["I"], r["L"], r["M"]) == (2, 4, {"S": 0, "P": 2, "O": 3})  # reference golden
    with pytest.raises(ValueError, match="no sm_100a realization"):
        twfa.Plan(prob, r["solution_json"])


def test_malformed_problem_is_rejected(twfa):
    _, sol = twfa.load_schedule("fa_fwd")
    with pytest.raises(ValueError):
        twfa.Plan("{not json", sol)
    with pytest.raises(ValueError, match="unknown key"):
        twfa.Plan(json.dumps({"machine": {}, "graph": {}, "extra": 1}), sol)


def test_s_ring_depth_from_pv_s_edge(twfa):
    """The double-buffered-S problem (PV_k -> S_k with delta 2) lowers to a
    2-deep S ring of 64-key tiles with the 4-deep K/V rings its solution
    streams; any other delta cannot be realized in 512 TMEM columns."""
    prob, sol = twfa.load_schedule("fa_fwd_ring2")
    d = twfa.Plan(prob, sol).describe()
    assert d["rings"] == {"K": 4, "V": 4, "S": 2} and d["kv_tile"] == 64
    p = json.loads(prob)
    for e in p["graph"]["edges"]:
        if e["src"] in ("PV0", "PV1") and e["dst"] == "S" + e["src"][2]:
            e["delta"] = 3
    with pytest.raises(ValueError, match="delta 1 or 2"):
        twfa.Plan(json.dumps(p), sol)


def test_fa_bwd_plan_roles_follow_the_solver(twfa):
    # the backward kernel's roles are the solver's warp assignment
    prob, sol = twfa.load_schedule("fa_bwd")
    s = json.loads(sol)
    d = twfa.Plan(prob, sol).describe()
    assert d["family"] == "fa_bwd"
    assert d["warpgroups"] == {"exp": s["A"]["EXB"], "ds": s["A"]["DS"], "dq_reduce": s["A"]["RD"]}
    assert d["p_transfer"].startswith("registers" if s["A"]["EXB"] == s["A"]["DS"] else "tensor memory")
    assert d["mma_warp"] == s["A"]["ST"] and d["load_warp"] == s["A"]["LDQ"]
    mma = d["warp_programs"][str(d["mma_warp"])]
    tc = [v for v in mma if v in ("ST", "DP", "DV", "DK", "DQ")]
    # issue order = slot order (M mod I) of the solution
    assert tc == sorted(tc, key=lambda v: s["M"][v] % s["I"])
    # the later reader of Q_i (ST, DK) / dO_i (DP, DV) releases the ring slot
    later = lambda a, b: a if s["M"][a] > s["M"][b] else b  # noqa: E731
    assert sorted(d["ring_release"]) == sorted([later("ST", "DK"), later("DP", "DV")])


@pytest.mark.parametrize("mutate,msg", [
    (lambda s: s["A"].update(DS=s["A"]["RD"]), "spill|own warpgroup"),
    (lambda s: s["A"].update(DQ=14), "variable_latency|issue from one warp"),
    (lambda s: s["A"].update(RD=12), "variable_latency|cannot be inside"),
    (lambda s: s["M"].update(DS=s["M"]["EXB"]), "dependence"),
])
def test_fa_bwd_unrealizable_solutions_are_rejected(twfa, mutate, msg):
    prob, sol = twfa.load_schedule("fa_bwd")
    s = json.loads(sol)
    mutate(s)
    with pytest.raises(ValueError, match=msg):
        twfa.Plan(prob, json.dumps(s))


def test_tile_makespan_formula_matches_reference_simulate(twfa, ws):
    # bench.py predicts a work tile's makespan as (N - 1) I + L units: the
    # reference's pipelined replay (simulate_pipeline, sim.cpp:371-466)
    prob, sol = twfa.load_schedule("fa_fwd")
    s = json.loads(sol)
    for n in (2, 3, 17, 64):  # the replay needs at least `copies` iterations
        assert ws.simulate(prob, sol, n)["cycles"] == (n - 1) * s["I"] + s["L"]


def test_fa_bwd_pp_plan_roles_follow_the_solver(twfa):
    """Two 64-query sub-tiles: EXB_k / DS_k fused on the solver's warpgroup of
    sub-tile k, RD_k on its own, all tensor-core ops on one warp in slot
    order, and the last reader of Q_i (dO_i) in issue order releases the slot."""
    prob, sol = twfa.load_schedule("fa_bwd_pp")
    s = json.loads(sol)
    d = twfa.Plan(prob, sol).describe()
    assert d["family"] == "fa_bwd" and d["num_tiles"] == 2
    assert d["warpgroups"] == {"exp_ds0": s["A"]["EXB0"], "exp_ds1": s["A"]["EXB1"],
                               "dq_reduce0": s["A"]["RD0"], "dq_reduce1": s["A"]["RD1"]}
    for k in (0, 1):
        assert s["A"][f"DS{k}"] == s["A"][f"EXB{k}"]
    mma = d["warp_programs"][str(d["mma_warp"])]
    tc = [v for v in mma if not v.startswith("LD")]
    assert sorted(tc) == sorted(f"{op}{k}" for op in ("ST", "DP", "DV", "DK", "DQ") for k in (0, 1))
    assert tc == sorted(tc, key=lambda v: (s["M"][v] // s["I"], s["M"][v] % s["I"]))
    last = lambda ids: max(ids, key=lambda v: (s["M"][v] // s["I"], mma.index(v)))  # noqa: E731
    assert sorted(d["ring_release"]) == sorted([last(["ST0", "ST1", "DK0", "DK1"]),
                                                last(["DP0", "DP1", "DV0", "DV1"])])


@pytest.mark.parametrize("mutate,msg", [
    (lambda s: s["A"].update(DS0=s["A"]["RD0"]), "spill|share a warpgroup"),
    (lambda s: s["A"].update(DQ1=14), "variable_latency|issue from one warp"),
    (lambda s: s["A"].update(RD1=s["A"]["EXB1"]), "register|own|spill"),
    (lambda s: s["M"].update(DS0=s["M"]["EXB0"]), "dependence"),
])
def test_fa_bwd_pp_unrealizable_solutions_are_rejected(twfa, mutate, msg):
    prob, sol = twfa.load_schedule("fa_bwd_pp")
    s = json.loads(sol)
    mutate(s)
    with pytest.raises(ValueError, match=msg):
        twfa.Plan(prob, json.dumps(s))


def test_fa_bwd_pp_without_aliasing_edges_is_rejected(twfa):
    # the kernel relies on the graph's tensor-memory / shared-memory aliasing edges
    prob, sol = twfa.load_schedule("fa_bwd_pp")
    p = json.loads(prob)
    p["graph"]["edges"] = [e for e in p["graph"]["edges"] if not (e["src"] == "RD0" and e["dst"] == "ST0")]
    with pytest.raises(ValueError, match="aliasing edge|dependence|validate"):
        twfa.Plan(json.dumps(p), sol)
