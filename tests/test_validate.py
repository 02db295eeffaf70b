"""The schedule checker libtwfa runs at twfa_plan_create against the
reference's own: validate_program (/root/reference/proj/src/sim.cpp:79-311)
over expand_solution's tables (sim.cpp:57-77) of the reconstructed solution
(cli.cpp:161-168), as the reference's Python binding returns it
(bindings/module.cpp:176-184). libtwfa restates the checker in C++
(lowering.cpp: validate_schedule); here both run on the committed schedules
and on seeded mutations of them (moved issue cycles, moved / misaligned warp
ranges, shrunk tensor memory and register limits), and must report the same
(family, message) list in the same order -- or both reject the documents."""
import copy
import glob
import json
import os
import random
import sys
import zlib

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCHED = os.path.join(ROOT, "paper_2512_18134_b200", "schedules")


@pytest.fixture(scope="module")
def ws():
    sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))
    try:
        import _weftsched
    except ImportError:
        pytest.skip("oracle/_ref not built")
    return _weftsched


def committed():
    out = []
    for f in sorted(glob.glob(os.path.join(SCHED, "*.solution.json"))):
        name = os.path.basename(f)[: -len(".solution.json")]
        out.append((name, open(os.path.join(SCHED, name + ".json")).read(), open(f).read()))
    for f in sorted(glob.glob(os.path.join(SCHED, "experiments", "*.solution.json"))):
        name = os.path.basename(f)[: -len(".solution.json")]
        pf = f[: -len(".solution.json")] + ".problem"
        prob = open(pf).read().strip() if os.path.exists(pf) else "fa_fwd"
        out.append((name, open(os.path.join(SCHED, prob + ".json")).read(), open(f).read()))
    return out


def ref_fixture_docs():
    """The reference's own data problems with the solutions its tests expect
    (tests/golden/ref_fixtures.json, from the internal solver)."""
    data = "/root/reference/proj/data"
    if not os.path.isdir(data):
        return []
    fx = json.load(open(os.path.join(ROOT, "tests", "golden", "ref_fixtures.json")))
    out = []
    for name, e in sorted(fx.items()):
        p = os.path.join(data, name + ".json")
        if os.path.exists(p):
            sol = {"I": e["I"], "L": e["L"], "M": e["M"], "A": e["A"]}
            out.append((name, open(p).read(), json.dumps(sol)))
    return out


def both(twfa, ws, prob, sol):
    """(ours, reference): the violation list, or the exception class name."""
    try:
        mine = [list(x) for x in twfa.validate(prob, sol)]
    except ValueError:
        mine = "ValueError"
    try:
        ref = [list(x) for x in ws.validate(prob, sol)]
    except (ValueError, RuntimeError):
        ref = "ValueError"
    return mine, ref


@pytest.mark.parametrize("name,prob,sol", committed(), ids=[c[0] for c in committed()])
def test_committed_schedules_are_exact_for_both_checkers(twfa, ws, name, prob, sol):
    mine, ref = both(twfa, ws, prob, sol)
    assert mine == ref == []


def test_reference_fixture_solutions_match(twfa, ws):
    docs = ref_fixture_docs()
    if not docs:
        pytest.skip("/root/reference not present")
    for name, prob, sol in docs:
        mine, ref = both(twfa, ws, prob, sol)
        assert mine == ref, name


def mutations(prob, sol, rng, n):
    p0, s0 = json.loads(prob), json.loads(sol)
    nodes = [nd["id"] for nd in p0["graph"]["nodes"]]
    nw = p0["machine"]["num_warps"]
    for _ in range(n):
        p, s = copy.deepcopy(p0), copy.deepcopy(s0)
        kind = rng.choice(["M", "M", "M2", "A", "A", "mem", "reg", "ML"])
        if kind in ("M", "M2"):
            for v in rng.sample(nodes, 1 if kind == "M" else 2):
                s["M"][v] = max(0, s["M"][v] + rng.choice([-3, -2, -1, 1, 2, 3]))
        elif kind == "ML":  # a different interval / length with the same M
            s["I"] = max(1, s["I"] + rng.choice([-2, -1, 1]))
            s["L"] = max(1, s["L"] + rng.choice([-1, 0, 1, 2]))
        elif kind == "A":
            v = rng.choice(nodes)
            s.setdefault("A", {})[v] = rng.randrange(-1, nw + 1)
        elif kind == "mem" and p["machine"].get("memories"):
            m = rng.choice(p["machine"]["memories"])
            m["capacity"] = max(0, m["capacity"] // rng.choice([2, 4]))
        elif kind == "reg":
            p["machine"]["reg_limit"] = rng.choice([1, 32, 64, 100, 128])
        yield json.dumps(p), json.dumps(s)


@pytest.mark.parametrize("name,prob,sol", committed()[:12], ids=[c[0] for c in committed()[:12]])
def test_mutated_schedules_match_reference_checker(twfa, ws, name, prob, sol):
    rng = random.Random(zlib.crc32(name.encode()))
    nonempty = 0
    for p, s in mutations(prob, sol, rng, 40):
        mine, ref = both(twfa, ws, p, s)
        assert mine == ref, (name, p, s)
        nonempty += isinstance(ref, list) and len(ref) > 0
    assert nonempty > 0  # the mutations do reach the checker


def test_plan_create_rejects_what_the_checker_rejects(twfa, ws):
    """The two cases the round-1 review named: two tensor-core ops in one
    cycle, tensor memory over its 512 columns."""
    prob, sol = twfa.load_schedule("fa_fwd")
    s = json.loads(sol)
    s["M"]["S0"] = s["M"]["S1"]  # S0 and S1 both on TC at the same cycles
    bad = json.dumps(s)
    assert any(f == "capacity" for f, _ in ws.validate(prob, bad))
    with pytest.raises(ValueError, match="validate_program.*capacity"):
        twfa.Plan(prob, bad)
    p = json.loads(prob)
    p["machine"]["memories"][0]["capacity"] = 320  # peak live tensor memory of the schedule is 384
    small = json.dumps(p)
    assert any(f == "memory" for f, _ in ws.validate(small, sol))
    with pytest.raises(ValueError, match="validate_program.*memory"):
        twfa.Plan(small, sol)


def test_validate_graph_restated(twfa):
    prob, sol = twfa.load_schedule("gemm_mainloop")
    p = json.loads(prob)
    # a zero-delta cycle MMA -> LDA -> MMA
    p["graph"]["edges"].append({"src": "MMA", "dst": "LDA", "d": 0})
    with pytest.raises(ValueError, match="zero-delta-cycle"):
        twfa.Plan(json.dumps(p), sol)
    p = json.loads(prob)
    p["graph"]["nodes"][0]["rrt"] = {p["machine"]["units"][0]["name"]: [5]}
    with pytest.raises(ValueError, match="rrt-exceeds-capacity"):
        twfa.Plan(json.dumps(p), sol)
