"""Pin the oracle before trusting it.

Schedule side: the reference built unmodified into oracle/_ref must reproduce
(1) the reference's OWN hard-coded test expectations for its fixtures, cited
per assertion, and (2) the committed golden outputs of tests/golden/
(make_golden.py). The committed FA / GEMM schedules must pass the reference's
validate_program and replay at the solver's steady rate 1/I.

Numerics side (parity unpinned by the reference, which has no attention
code): the C restatement must reproduce the committed fp64 fixtures.
"""
import json
import os
import sys

import numpy as np
import pytest

from tests import oracle_lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")
REF_DATA = "/root/reference/proj/data"


def golden(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


@pytest.fixture(scope="module")
def ws():
    sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))
    try:
        import _weftsched
    except ImportError:
        pytest.skip("oracle/_ref not built")
    return _weftsched


def test_goldens_match_reference_test_expectations():
    g = golden("ref_fixtures.json")
    a = g["attention_simple"]
    # cli_viz_test.cpp:146-166 and jointsolve_test.cpp:318-329
    assert (a["I"], a["L"]) == (2, 4)
    assert a["M"] == {"S": 0, "P": 2, "O": 3}
    assert a["A"] == {"S": 0, "P": 0, "O": 0}
    assert a["streaming_depths"] == {}
    assert a["search_report"] == [{"I": 1, "L": None, "outcome": "no_modulo_schedule"},
                                  {"I": 2, "L": 4, "outcome": "sat"}]
    # jointsolve_test.cpp:204-216 (blocking_sync_problem(1) == blocking_one_warp.json)
    b = g["blocking_one_warp"]
    assert b["search_report"] == [{"I": 1, "L": 3, "outcome": "unsat"}, {"I": 2, "L": 3, "outcome": "sat"}]
    assert b["streaming_depths"] == {"LOAD": 2}
    # jointsolve_test.cpp:301-316
    c = g["search_climb"]
    assert c["search_report"] == [{"I": 1, "L": None, "outcome": "no_modulo_schedule"},
                                  {"I": 2, "L": 2, "outcome": "unsat"}, {"I": 3, "L": 2, "outcome": "unsat"},
                                  {"I": 3, "L": 3, "outcome": "sat"}]
    assert c["streaming_depths"] == {}
    # codegen_test.cpp:59-89: the Fig. 1f steady state
    steady = a["listing"].split("steady_state:")[1].split("epilogue:")[0]
    for line in ("Sn = S()", "P = P(S)", "O = O(P, O[i-1])", "S = Sn"):
        assert line in steady
    for e in g.values():
        assert e["validate"] == []


def test_reference_replay_counts(ws):
    """sim_test.cpp:90-115: Fig. 1 at I=2 replays 4 iterations in 10 cycles
    (rate 2/5) and 10 in 22 (5/11), steady 1/2 -- through the oracle build."""
    sol = json.dumps(golden("ref_fixtures.json")["attention_simple"]["solution"])
    if not os.path.isdir(REF_DATA):
        pytest.skip("reference fixtures not present (GPU box)")
    prob = open(os.path.join(REF_DATA, "attention_simple.json")).read()
    r4, r10 = ws.simulate(prob, sol, 4), ws.simulate(prob, sol, 10)
    assert (r4["cycles"], tuple(r4["throughput"]), tuple(r4["steady"])) == (10, (2, 5), (1, 2))
    assert (r10["cycles"], tuple(r10["throughput"]), tuple(r10["steady"])) == (22, (5, 11), (1, 2))


def test_oracle_build_reproduces_goldens(ws):
    if not os.path.isdir(REF_DATA):
        pytest.skip("reference fixtures not present (GPU box)")
    g = golden("ref_fixtures.json")
    for name, e in g.items():
        prob = open(os.path.join(REF_DATA, name + ".json")).read()
        r = ws.joint(prob, 0, 2, "")
        assert r["status"] == e["status"]
        assert r["search_report"] == e["search_report"]
        assert (r["I"], r["L"], r["M"], r["A"]) == (e["I"], e["L"], e["M"], e["A"])
        assert ws.codegen(prob, r["solution_json"], "text") == e["listing"]
        sim = ws.simulate(prob, r["solution_json"], 16)
        assert sim["cycles"] == e["sim16"]["cycles"]


@pytest.mark.parametrize("name", sorted(golden("fa_schedules.json")))
def test_committed_schedules_validate_and_replay(ws, twfa, name):
    prob, sol = twfa.load_schedule(name)
    e = golden("fa_schedules.json")[name]
    assert ws.validate(prob, sol) == [] == e["validate"]
    sim = ws.simulate(prob, sol, 64)
    I = json.loads(sol)["I"]
    assert tuple(sim["steady"]) == (1, I)
    assert sim["cycles"] == e["sim64_cycles"]


def test_lowering_rejects_reference_toy_fixtures(twfa):
    """The reference's fixtures are not the FA / GEMM loops: the executor
    must refuse them as a domain error (ValueError), never guess a kernel."""
    if not os.path.isdir(REF_DATA):
        pytest.skip("reference fixtures not present (GPU box)")
    g = golden("ref_fixtures.json")
    for name in ("attention_simple", "wide_attention_block"):
        prob = open(os.path.join(REF_DATA, name + ".json")).read()
        with pytest.raises(ValueError, match="no sm_100a realization|neither"):
            twfa.Plan(prob, json.dumps(g[name]["solution"]))


@pytest.mark.parametrize("causal", [False, True])
def test_c_oracle_matches_fp64_fixture(causal):
    z = np.load(os.path.join(GOLD, "attention_small.npz"))
    tag = "causal" if causal else "full"
    o, lse = oracle_lib.attention(z["q"], z["k"], z["v"], causal=causal)
    assert np.abs(o - z["o_" + tag]).max() < 2e-6
    assert np.abs(lse - z["lse_" + tag]).max() < 2e-6
    oo, lo = oracle_lib.attention(z["q"], z["k"], z["v"], causal=causal, online=True, tile=128)
    assert np.abs(oo - z["o_" + tag]).max() < 2e-5
    assert np.abs(lo - z["lse_" + tag]).max() < 2e-5
