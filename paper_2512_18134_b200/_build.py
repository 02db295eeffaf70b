"""Build libtwfa.so in-tree (sm_100a only) with explicit nvcc/g++ commands.

The library is the product: the CUDA kernels (fa_fwd_sm100.cu, gemm_sm100.cu),
the schedule lowering (lowering.cpp) and the extern "C" boundary (capi.cpp,
include/twfa.h). No torch types cross it.
"""
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "_obj")
LIB = os.path.join(PKG, "libtwfa.so")
HOST_TOOL = os.path.join(PKG, "twfa-run")
GEN_TOOL = os.path.join(PKG, "twfa-gen")
GEN_INC = os.path.join(CSRC, "gen", "fa_plans.inc")
SCHED = os.path.join(PKG, "schedules")


def specializations():
    """(identifier, problem, solution) of every committed FA schedule: each
    gets a build-time specialized kernel (csrc/gen_main.cpp)."""
    out = []
    for f in sorted(os.listdir(SCHED)):
        if f.endswith(".solution.json") and f.startswith("fa_fwd"):
            name = f[: -len(".solution.json")]
            out.append((name, os.path.join(SCHED, name + ".json"), os.path.join(SCHED, f)))
    exp = os.path.join(SCHED, "experiments")
    if os.path.isdir(exp):
        for f in sorted(os.listdir(exp)):
            if f.endswith(".solution.json"):
                name = f[: -len(".solution.json")]
                # hand-edited assignments (not solver output); <name>.problem names
                # the problem they apply to (default fa_fwd)
                pf = os.path.join(exp, name + ".problem")
                prob = open(pf).read().strip() if os.path.exists(pf) else "fa_fwd"
                out.append((name, os.path.join(SCHED, prob + ".json"), os.path.join(exp, f)))
    only = os.environ.get("TWFA_SPECIALIZE")  # comma list: limit (experiment builds)
    if only is not None:
        keep = set(only.split(",")) - {""}
        out = [e for e in out if e[0] in keep]
    return out


def generate_plans(gen_root, verbose=False):
    """twfa-gen: lowering.cpp + gen_main.cpp on the host compiler, then the
    committed schedules -> <gen_root>/gen/: fa_plans.inc (compile-time
    TwfaDevicePlans), one fa_spec_<id>.cu per specialization, and their
    launcher declarations."""
    inc = ["-I" + CSRC, "-I" + json_include()]
    tool = os.path.join(gen_root, "twfa-gen") if gen_root != CSRC else GEN_TOOL
    run([host_cxx(), "-std=c++20", "-O1", "-Wall", os.path.join(CSRC, "lowering.cpp"), os.path.join(CSRC, "gen_main.cpp"),
         *inc, "-o", tool], verbose)
    gen = os.path.join(gen_root, "gen")
    if os.path.isdir(gen):
        for f in os.listdir(gen):
            os.remove(os.path.join(gen, f))
    os.makedirs(gen, exist_ok=True)
    args = [tool, os.path.join(gen, "fa_plans.inc")]
    for name, prob, sol in specializations():
        args += [name, prob, sol]
    run(args, verbose)
    return GEN_INC

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CUDA_HOME = os.path.dirname(os.path.dirname(NVCC))
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def json_include():
    import sysconfig
    p = os.path.join(sysconfig.get_paths()["purelib"], "include", "cudnn_frontend", "thirdparty", "nlohmann")
    if not os.path.exists(os.path.join(p, "json.hpp")):
        raise RuntimeError("nlohmann/json.hpp not found at " + p)
    return p


def host_cxx():
    # the /opt/gcc wrapper works for plain C++; prefer the system compiler
    return "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"


def run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("build step failed: " + " ".join(cmd[:3]))
    return r.stdout + r.stderr


def sources(gen_root=CSRC):
    gen = os.path.join(gen_root, "gen")
    specs = sorted(os.path.join(gen, f) for f in os.listdir(gen) if f.startswith("fa_spec_") and f.endswith(".cu")) \
        if os.path.isdir(gen) else []
    cu = [os.path.join(CSRC, f) for f in ("fa_fwd_sm100.cu", "fa_bwd_sm100.cu", "fa_bwd_pp_sm100.cu",
                                          "gemm_sm100.cu")] + specs
    cpp = [os.path.join(CSRC, f) for f in ("lowering.cpp", "capi.cpp")]
    return cu, cpp


def stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f != "gen"] + [
        os.path.join(ROOT, "include", "twfa.h"), os.path.join(PKG, "host", "twfa_run.cpp"),
        os.path.join(PKG, "host", "twfa_pybind.cpp")]
    deps += [p for _, a, b in specializations() for p in (a, b)]
    if not os.path.exists(HOST_TOOL):
        return True
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False, ptxas_info=False, defines=(), out=None):
    """Compile libtwfa.so (or, with `defines`/`out`, a kernel variant for experiments)."""
    lib = out or LIB
    if not force and not defines and out is None and not stale():
        return LIB
    obj_dir = OBJ if not defines else os.path.join(OBJ, "v_" + "_".join(d.replace("=", "") for d in defines))
    os.makedirs(obj_dir, exist_ok=True)
    # variant builds keep their generated specializations next to their objects
    gen_root = CSRC if (out is None and not defines) else obj_dir
    generate_plans(gen_root, verbose)
    cu, cpp = sources(gen_root)
    inc = ["-I" + gen_root, "-I" + CSRC, "-I" + os.path.join(ROOT, "include"), "-I" + json_include()]
    objs = []
    log = ""
    cmds = []
    for src in cu:
        obj = os.path.join(obj_dir, os.path.basename(src) + ".o")
        cmds.append([NVCC, *ARCH, "-std=c++20", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-c", src, "-o", obj, *inc,
                     "--use_fast_math", "-Xptxas", "-v" if ptxas_info else "-O3", *["-D" + d for d in defines]])
        objs.append(obj)
    # the translation units are independent: compile them concurrently
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(len(cmds), os.cpu_count() or 4)) as ex:
        for out_text in ex.map(lambda c: run(c, verbose), cmds):
            log += out_text
    for src in cpp:
        obj = os.path.join(obj_dir, os.path.basename(src) + ".o")
        cmd = [host_cxx(), "-std=c++17", "-O2", "-fPIC", "-Wall", "-c", src, "-o", obj, *inc,
               "-I" + os.path.join(CUDA_HOME, "include")]
        log += run(cmd, verbose)
        objs.append(obj)
    tmp = lib + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart"]
    log += run(cmd, verbose)
    shutil.move(tmp, lib)
    if out is None and not defines:
        build_host_tool(verbose)
        build_pybind(verbose)
    if ptxas_info:
        print(log)
    return lib


def build_pybind(verbose=False):
    """_twfa: the pybind11 module over the C ABI (host/twfa_pybind.cpp), the
    counterpart of the reference's _weftsched; rpath $ORIGIN to libtwfa.so."""
    import sysconfig
    import pybind11
    ext = sysconfig.get_config_var("EXT_SUFFIX")
    out = os.path.join(PKG, "_twfa" + ext)
    cmd = [host_cxx(), "-std=c++17", "-O2", "-Wall", "-shared", "-fPIC", os.path.join(PKG, "host", "twfa_pybind.cpp"),
           "-I" + os.path.join(ROOT, "include"), "-I" + sysconfig.get_paths()["include"], "-I" + pybind11.get_include(),
           "-L" + PKG, "-ltwfa", "-Wl,-rpath,$ORIGIN", "-o", out]
    run(cmd, verbose)
    return out


def build_host_tool(verbose=False):
    """twfa-run: the C++ host program over the C ABI (host/twfa_run.cpp),
    linked against the in-tree libtwfa.so (rpath $ORIGIN)."""
    src = os.path.join(PKG, "host", "twfa_run.cpp")
    cmd = [host_cxx(), "-std=c++17", "-O2", "-Wall", "-Wextra", src, "-I" + os.path.join(ROOT, "include"),
           "-L" + PKG, "-ltwfa", "-Wl,-rpath,$ORIGIN", "-o", HOST_TOOL]
    run(cmd, verbose)
    return HOST_TOOL


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a[6:] for a in sys.argv[1:] if a.startswith("--out=")]
    build(force="--force" in sys.argv, verbose=True, ptxas_info="--ptxas" in sys.argv, defines=defs,
          out=outs[0] if outs else None)
