"""B200-native executor for Twill (arXiv 2512.18134) schedules.

The reference (`weftsched`) turns a loop dependence graph + machine model into
a modulo schedule with a warp assignment; its Python surface takes and returns
the same JSON documents as its CLI (reference: proj/bindings/module.cpp:219-249,
proj/python/weftsched/__init__.py). This package keeps that convention: a plan
is created from the problem JSON and the solution JSON `weftsched.joint`
returns (`solution_json`), and then executes the scheduled loop on sm_100a.

    from paper_2512_18134_b200 import Plan, fa_fwd, load_schedule
    plan = Plan(*load_schedule("fa_fwd"))
    o, lse = fa_fwd(plan, q, k, v, causal=False, return_lse=True)

Everything below is a thin ctypes layer over libtwfa.so (include/twfa.h); the
only compute path is the CUDA kernels in that library. There is no CPU
fallback: without the library or a GPU, calls raise.
"""
import ctypes
import json
import math
import os

__all__ = [
    "Plan",
    "TwfaError",
    "fa_fwd",
    "fa_fwd_host",
    "gemm",
    "lib",
    "load_schedule",
    "schedule_dir",
    "validate",
]

_PKG = os.path.dirname(os.path.abspath(__file__))
# TWFA_LIB selects an alternative in-tree build (kernel-variant experiments)
_LIB_PATH = os.environ.get("TWFA_LIB") or os.path.join(_PKG, "libtwfa.so")
_lib = None


class TwfaError(RuntimeError):
    """CUDA-side failure (return code 3)."""


def lib():
    """Load libtwfa.so (built in-tree by __graft_entry__.build())."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise ImportError(f"{_LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(_LIB_PATH)
        vp, i32, f32, sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_float, ctypes.c_size_t
        L.twfa_abi_version.restype = i32
        L.twfa_last_error.restype = ctypes.c_char_p
        L.twfa_plan_create.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.POINTER(vp)]
        L.twfa_plan_destroy.argtypes = [vp]
        L.twfa_schedule_validate.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p, sz,
                                             ctypes.POINTER(sz)]
        L.twfa_plan_describe.argtypes = [vp, ctypes.c_char_p, sz, ctypes.POINTER(sz)]
        L.twfa_plan_raw.argtypes = [vp, vp, sz, ctypes.POINTER(sz)]
        L.twfa_fa_fwd.argtypes = [vp, vp, vp, vp, vp, vp, i32, i32, i32, i32, i32, f32, vp]
        L.twfa_fa_fwd_traced.argtypes = [vp, vp, vp, vp, vp, vp, i32, i32, i32, i32, i32, f32, vp,
                                         ctypes.c_uint32, vp]
        L.twfa_fa_fwd_host.argtypes = [vp, vp, vp, vp, vp, vp, i32, i32, i32, i32, i32, f32]
        L.twfa_gemm.argtypes = [vp, vp, vp, vp, i32, i32, i32, vp]
        L.twfa_grid_size.argtypes = [ctypes.POINTER(i32)]
        L.twfa_fa_bwd_workspace_size.argtypes = [i32, i32, i32, i32, ctypes.POINTER(sz)]
        L.twfa_fa_bwd.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, sz, i32, i32, i32, i32, i32, f32, vp]
        L.twfa_fa_bwd_traced.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, sz, i32, i32, i32, i32, i32, f32,
                                         vp, ctypes.c_uint32, vp]
        for name in ("twfa_schedule_validate", "twfa_plan_create", "twfa_plan_describe", "twfa_plan_raw", "twfa_fa_fwd",
                     "twfa_fa_fwd_traced", "twfa_fa_fwd_host", "twfa_gemm", "twfa_grid_size",
                     "twfa_fa_bwd_workspace_size", "twfa_fa_bwd", "twfa_fa_bwd_traced"):
            getattr(L, name).restype = i32
        _lib = L
    return _lib


def _check(rc):
    if rc == 0:
        return
    msg = lib().twfa_last_error().decode()
    # reference convention: malformed documents / arguments surface as
    # ValueError (std::invalid_argument through pybind, test_smoke.py:80-82)
    if rc in (1, 2):
        raise ValueError(msg)
    raise TwfaError(msg)


def schedule_dir():
    return os.path.join(_PKG, "schedules")


def load_schedule(name):
    """(problem_json, solution_json) texts of a committed golden schedule."""
    d = schedule_dir()
    with open(os.path.join(d, name + ".json")) as f:
        prob = f.read()
    with open(os.path.join(d, name + ".solution.json")) as f:
        sol = f.read()
    return prob, sol


def validate(problem_json, solution_json):
    """The reference checker (validate_program, sim.cpp:79-311) restated in
    libtwfa: [(family, message), ...], empty when the schedule is exact."""
    need = ctypes.c_size_t()
    p, q = problem_json.encode(), solution_json.encode()
    _check(lib().twfa_schedule_validate(p, q, None, 0, ctypes.byref(need)))
    buf = ctypes.create_string_buffer(need.value)
    _check(lib().twfa_schedule_validate(p, q, buf, need.value, ctypes.byref(need)))
    return [tuple(x) for x in json.loads(buf.value.decode())]


class Plan:
    """A solved schedule lowered for the B200 kernels (twfa_plan_create)."""

    def __init__(self, problem_json, solution_json):
        h = ctypes.c_void_p()
        _check(lib().twfa_plan_create(problem_json.encode(), solution_json.encode(), ctypes.byref(h)))
        self._h = h

    @property
    def handle(self):
        return self._h

    def describe(self):
        need = ctypes.c_size_t()
        _check(lib().twfa_plan_describe(self._h, None, 0, ctypes.byref(need)))
        buf = ctypes.create_string_buffer(need.value)
        _check(lib().twfa_plan_describe(self._h, buf, need.value, ctypes.byref(need)))
        return json.loads(buf.value.decode())

    def raw(self):
        need = ctypes.c_size_t()
        _check(lib().twfa_plan_raw(self._h, None, 0, ctypes.byref(need)))
        buf = ctypes.create_string_buffer(need.value)
        _check(lib().twfa_plan_raw(self._h, buf, need.value, ctypes.byref(need)))
        return buf.raw

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            _lib.twfa_plan_destroy(h)
            self._h = None


def _stream_ptr(t):
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


def fa_fwd(plan, q, k, v, causal=False, softmax_scale=None, return_lse=False, out=None, trace=None,
           trace_cap=0):
    """FA forward on the current CUDA stream. q, k, v: [B, H, S, 128] bf16 CUDA
    tensors (contiguous). Returns o (and lse [B, H, S] fp32 if return_lse)."""
    import torch
    if q.dtype != torch.bfloat16 or k.dtype != torch.bfloat16 or v.dtype != torch.bfloat16:
        raise ValueError("q, k, v must be bf16")
    if not (q.is_cuda and k.is_cuda and v.is_cuda):
        raise ValueError("q, k, v must be CUDA tensors")
    if q.shape != k.shape or q.shape != v.shape or q.dim() != 4:
        raise ValueError("q, k, v must share shape [B, H, S, D]")
    q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
    B, H, S, D = q.shape
    scale = float(softmax_scale) if softmax_scale is not None else 1.0 / math.sqrt(D)
    if out is not None:
        # the C side encodes O's tensor map as a contiguous bf16 [B, H, S, 128]
        if out.shape != q.shape or out.dtype != torch.bfloat16 or out.device != q.device or not out.is_contiguous():
            raise ValueError("out must be a contiguous bf16 tensor of q's shape on q's device")
    if k.device != q.device or v.device != q.device:
        raise ValueError("q, k, v must be on one device")
    o = out if out is not None else torch.empty_like(q)
    lse = torch.empty((B, H, S), device=q.device, dtype=torch.float32) if return_lse else None
    if trace is not None:
        need = plan.describe()["num_warps"] * int(trace_cap) * 8
        if trace.dtype not in (torch.int32, torch.uint32) or not trace.is_contiguous() or trace.device != q.device \
                or trace.numel() < need or trace_cap < 2:
            raise ValueError(f"trace must be a contiguous int32 tensor on q's device with >= num_warps * trace_cap "
                             f"* 8 = {need} elements (trace_cap >= 2)")
    args = (plan.handle, ctypes.c_void_p(q.data_ptr()), ctypes.c_void_p(k.data_ptr()),
            ctypes.c_void_p(v.data_ptr()), ctypes.c_void_p(o.data_ptr()),
            ctypes.c_void_p(lse.data_ptr()) if lse is not None else None,
            B, H, S, D, int(bool(causal)), scale)
    with torch.cuda.device(q.device):
        if trace is not None:
            _check(lib().twfa_fa_fwd_traced(*args, ctypes.c_void_p(trace.data_ptr()), trace_cap, _stream_ptr(q)))
        else:
            _check(lib().twfa_fa_fwd(*args, _stream_ptr(q)))
    return (o, lse) if return_lse else o


def fa_fwd_host(plan, q, k, v, causal=False, softmax_scale=None, return_lse=False, out=None, lse_out=None):
    """Host-buffer form (twfa_fa_fwd_host): numpy uint16 arrays of bf16 bit
    patterns, [B, H, S, 128]. Synchronous; the pairs stream through the
    library's chunked copy/compute pipeline. Page-locked buffers (e.g. numpy
    views of torch pin_memory tensors) are DMA'd directly -- pass `out` (and
    `lse_out`) page-locked too to keep the whole call on that path."""
    import numpy as np
    q, k, v = (np.ascontiguousarray(x, dtype=np.uint16) for x in (q, k, v))
    if q.shape != k.shape or q.shape != v.shape or q.ndim != 4:
        raise ValueError("q, k, v must share shape [B, H, S, D]")
    B, H, S, D = q.shape
    scale = float(softmax_scale) if softmax_scale is not None else 1.0 / math.sqrt(D)
    if out is not None and (out.shape != q.shape or out.dtype != np.uint16 or not out.flags.c_contiguous):
        raise ValueError("out must be a contiguous uint16 array of q's shape")
    o = out if out is not None else np.empty_like(q)
    if lse_out is not None and (lse_out.shape != (B, H, S) or lse_out.dtype != np.float32
                                or not lse_out.flags.c_contiguous):
        raise ValueError("lse_out must be a contiguous float32 [B, H, S] array")
    lse = lse_out if lse_out is not None else (np.empty((B, H, S), dtype=np.float32) if return_lse else None)
    p = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    _check(lib().twfa_fa_fwd_host(plan.handle, p(q), p(k), p(v), p(o), p(lse) if lse is not None else None,
                                  B, H, S, D, int(bool(causal)), scale))
    return (o, lse) if (return_lse or lse_out is not None) else o


def fa_bwd(plan, q, k, v, o, dout, lse, causal=False, softmax_scale=None, workspace=None, trace=None,
           trace_cap=0):
    """FA backward on the current CUDA stream (plan from an FA-backward
    schedule, e.g. load_schedule("fa_bwd")). q, k, v, o, dout: [B, H, S, 128]
    bf16 CUDA tensors; lse: [B, H, S] fp32 from fa_fwd(..., return_lse=True).
    Returns (dq, dk, dv) bf16."""
    import torch
    ts = (q, k, v, o, dout)
    if any(t.dtype != torch.bfloat16 for t in ts):
        raise ValueError("q, k, v, o, dout must be bf16")
    if any(not t.is_cuda for t in ts) or not lse.is_cuda:
        raise ValueError("inputs must be CUDA tensors")
    if any(t.shape != q.shape for t in ts) or q.dim() != 4:
        raise ValueError("q, k, v, o, dout must share shape [B, H, S, D]")
    q, k, v, o, dout = (t.contiguous() for t in ts)
    B, H, S, D = q.shape
    if lse.dtype != torch.float32 or tuple(lse.shape) != (B, H, S):
        raise ValueError("lse must be fp32 [B, H, S]")
    lse = lse.contiguous()
    scale = float(softmax_scale) if softmax_scale is not None else 1.0 / math.sqrt(D)
    need = ctypes.c_size_t()
    _check(lib().twfa_fa_bwd_workspace_size(B, H, S, D, ctypes.byref(need)))
    if workspace is None or workspace.numel() * workspace.element_size() < need.value:
        workspace = torch.empty(need.value, device=q.device, dtype=torch.uint8)
    dq, dk, dv = (torch.empty_like(q) for _ in range(3))
    if any(t.device != q.device for t in ts) or lse.device != q.device:
        raise ValueError("inputs must be on one device")
    ptr = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    with torch.cuda.device(q.device):
        args = (plan.handle, ptr(q), ptr(k), ptr(v), ptr(o), ptr(dout), ptr(lse), ptr(dq), ptr(dk), ptr(dv),
                ptr(workspace), need.value, B, H, S, D, int(bool(causal)), scale)
        if trace is not None:
            nw = plan.describe()["num_warps"]
            if trace.dtype != torch.int32 or not trace.is_contiguous() or trace.numel() < nw * int(trace_cap) * 8:
                raise ValueError("trace must be a contiguous int32 tensor of >= num_warps * trace_cap * 8 elements")
            _check(lib().twfa_fa_bwd_traced(*args, ptr(trace), trace_cap, _stream_ptr(q)))
        else:
            _check(lib().twfa_fa_bwd(*args, _stream_ptr(q)))
    return dq, dk, dv


def gemm(plan, a, b, out=None):
    """C = A @ B^T with A [M, K], B [N, K] bf16 CUDA tensors."""
    import torch
    if a.dtype != torch.bfloat16 or b.dtype != torch.bfloat16:
        raise ValueError("a, b must be bf16")
    a, b = a.contiguous(), b.contiguous()
    M, K = a.shape
    N = b.shape[0]
    if b.shape[1] != K:
        raise ValueError("a and b must share K")
    if b.device != a.device:
        raise ValueError("a and b must be on one device")
    if out is not None and (tuple(out.shape) != (M, N) or out.dtype != torch.bfloat16 or out.device != a.device
                            or not out.is_contiguous()):
        raise ValueError("out must be a contiguous bf16 [M, N] tensor on a's device")
    c = out if out is not None else torch.empty((M, N), device=a.device, dtype=torch.bfloat16)
    with torch.cuda.device(a.device):
        _check(lib().twfa_gemm(plan.handle, ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(b.data_ptr()),
                               ctypes.c_void_p(c.data_ptr()), M, N, K, _stream_ptr(a)))
    return c
