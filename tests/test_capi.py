"""The C-ABI library (libtwfa.so) loads and exports every function declared in
include/twfa.h; argument / document errors come back as the reference's exit
codes (1 domain, 2 usage) with a message, without a GPU."""
import ctypes
import json
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    text = open(os.path.join(ROOT, "include", "twfa.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(twfa_[a-z_0-9]+)\s*\(", text)))


def test_every_declared_symbol_is_exported(twfa):
    lib = ctypes.CDLL(twfa._LIB_PATH)
    names = declared_functions()
    assert len(names) >= 10
    for n in names:
        assert hasattr(lib, n), n


def test_error_codes_and_messages(twfa):
    L = twfa.lib()
    h = ctypes.c_void_p()
    assert L.twfa_plan_create(b"{}", b"{}", ctypes.byref(h)) == 1
    assert b"machine" in L.twfa_last_error()
    assert L.twfa_plan_create(None, b"{}", ctypes.byref(h)) == 2
    prob, sol = twfa.load_schedule("gemm_mainloop")
    assert L.twfa_plan_create(prob.encode(), sol.encode(), ctypes.byref(h)) == 0
    assert L.twfa_last_error() == b""
    # an FA launch with a GEMM plan is a usage error, detected before any CUDA call
    rc = L.twfa_fa_fwd(h, None, None, None, None, None, 1, 1, 128, 128, 0, 1.0, None)
    assert rc == 2 and b"not an FA-forward plan" in L.twfa_last_error()
    rc = L.twfa_gemm(h, None, None, None, 100, 256, 64, None)
    assert rc == 2
    need = ctypes.c_size_t()
    assert L.twfa_plan_raw(h, None, 0, ctypes.byref(need)) == 0 and need.value > 0
    L.twfa_plan_destroy(h)
    assert L.twfa_abi_version() == 2


def test_plan_survives_threads(twfa):
    import threading
    prob, sol = twfa.load_schedule("fa_fwd")
    out = []

    def work():
        out.append(twfa.Plan(prob, sol).describe()["I"])

    ts = [threading.Thread(target=work) for _ in range(8)]
    [t.start() for t in ts]
    [t.join() for t in ts]
    assert out == [json.loads(sol)["I"]] * 8


def _host_tool(twfa):
    from paper_2512_18134_b200 import _build
    if not os.path.exists(_build.HOST_TOOL):
        _build.build_host_tool()
    return _build.HOST_TOOL


def test_host_tool_exit_codes(twfa):
    """twfa-run (the C++ host over the C ABI) follows the reference CLI's exit
    map (cli.cpp:462-471): 2 usage, 1 domain error, 0 ok."""
    import subprocess
    tool = _host_tool(twfa)
    d = twfa.schedule_dir()
    prob, sol = os.path.join(d, "fa_fwd.json"), os.path.join(d, "fa_fwd.solution.json")
    assert subprocess.run([tool, "fa", prob], capture_output=True).returncode == 2
    assert subprocess.run([tool, "bogus", prob, sol], capture_output=True).returncode == 2
    assert subprocess.run([tool, "fa", prob, sol, "--S", "x"], capture_output=True).returncode == 2
    r = subprocess.run([tool, "fa", prob, os.path.join(d, "gemm_mainloop.solution.json")], capture_output=True,
                       text=True)
    assert r.returncode == 1 and "unknown node" in r.stderr
    r = subprocess.run([tool, "describe", prob, sol], capture_output=True, text=True)
    assert r.returncode == 0
    assert json.loads(r.stdout)["I"] == json.loads(open(sol).read())["I"]


def _pybind(twfa):
    import importlib
    import sys
    from paper_2512_18134_b200 import _build
    pkg = os.path.dirname(_build.LIB)
    if not any(f.startswith("_twfa") for f in os.listdir(pkg)):
        _build.build_pybind()
    if pkg not in sys.path:
        sys.path.insert(0, pkg)
    return importlib.import_module("_twfa")


def test_pybind_module_mirrors_reference_conventions(twfa):
    """_twfa (pybind11 over the C ABI) is JSON in / dict out like the
    reference's _weftsched (module.cpp:219-249); bad documents raise
    ValueError (test_smoke.py:80-82)."""
    import pytest
    m = _pybind(twfa)
    prob, sol = twfa.load_schedule("fa_fwd")
    d = m.describe(prob, sol)
    assert d["I"] == json.loads(sol)["I"] and d == twfa.Plan(prob, sol).describe()
    with pytest.raises(ValueError, match="machine"):
        m.Plan("{}", "{}")
    with pytest.raises(ValueError, match="unknown solution key"):
        m.Plan(prob, json.dumps(dict(json.loads(sol), bogus=1)))
    assert m.validate(prob, sol) == []
    bad = json.loads(sol)
    bad["A"]["S0"] = 3
    assert [f for f, _ in m.validate(prob, json.dumps(bad))] == ["variable_latency"]


def test_fa_bwd_entry_points_check_arguments_without_a_gpu(twfa):
    L = twfa.lib()
    n = ctypes.c_size_t()
    assert L.twfa_fa_bwd_workspace_size(2, 4, 1000, 128, ctypes.byref(n)) == 0
    rows = 2 * 4 * 1000
    assert n.value == rows * 128 * 4 + rows * 4  # fp32 dQ accumulator + rowsum(dO * O)
    assert L.twfa_fa_bwd_workspace_size(1, 1, 128, 64, ctypes.byref(n)) == 2
    h = ctypes.c_void_p()
    prob, sol = twfa.load_schedule("fa_fwd")
    assert L.twfa_plan_create(prob.encode(), sol.encode(), ctypes.byref(h)) == 0
    args = [None] * 10 + [0, 1, 1, 128, 128, 0, ctypes.c_float(1.0), None]
    # a forward plan is a usage error, detected before any CUDA call
    assert L.twfa_fa_bwd(h, *args) == 2 and b"FA-backward plan" in L.twfa_last_error()
    assert L.twfa_fa_bwd(None, *args) == 2
    L.twfa_plan_destroy(h)
    prob, sol = twfa.load_schedule("fa_bwd")
    assert L.twfa_plan_create(prob.encode(), sol.encode(), ctypes.byref(h)) == 0
    assert L.twfa_fa_bwd(h, *args) == 2 and b"NULL" in L.twfa_last_error()  # q is NULL
    L.twfa_plan_destroy(h)
