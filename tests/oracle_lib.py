"""ctypes loader for the C oracle (oracle/_build/liboracle.so).

TEST INFRASTRUCTURE: the oracle is the checker, never the measured path.
"""
import ctypes
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "oracle", "_build", "liboracle.so")
_lib = None


def build():
    srcs = [os.path.join(ROOT, "oracle", f) for f in ("attention.c", "gemm.c", "oracle.h")]
    if os.path.exists(LIB) and all(os.path.getmtime(LIB) >= os.path.getmtime(s) for s in srcs):
        return LIB
    subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "lib"], check=True, capture_output=True)
    return LIB


def load():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB)
        vp, i32, f32 = ctypes.c_void_p, ctypes.c_int, ctypes.c_float
        L.oracle_attention.argtypes = [vp, vp, vp, vp, vp, i32, i32, i32, i32, i32, i32, f32, i32]
        L.oracle_attention_online.argtypes = [vp, vp, vp, vp, vp, i32, i32, i32, i32, i32, i32, f32, i32, i32]
        L.oracle_attention_bwd.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, vp, i32, i32, i32, i32, i32, f32, i32]
        L.oracle_gemm_tn.argtypes = [vp, vp, vp, i32, i32, i32, i32]
        L.oracle_round_bf16.argtypes = [vp, ctypes.c_int64]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def attention(q, k, v, causal=False, scale=None, online=False, tile=128, threads=0):
    """q: float32 [B, H, Sq, D]; k, v: [B, H, Sk, D] (queries = the first Sq
    positions). Returns (o, lse)."""
    L = load()
    q, k, v = (np.ascontiguousarray(x, dtype=np.float32) for x in (q, k, v))
    B, H, Sq, D = q.shape
    Sk = k.shape[2]
    scale = float(scale if scale is not None else 1.0 / np.sqrt(D))
    o = np.empty_like(q)
    lse = np.empty((B, H, Sq), dtype=np.float32)
    if online:
        L.oracle_attention_online(_p(q), _p(k), _p(v), _p(o), _p(lse), B, H, Sq, Sk, D, int(causal), scale, tile,
                                  threads)
    else:
        L.oracle_attention(_p(q), _p(k), _p(v), _p(o), _p(lse), B, H, Sq, Sk, D, int(causal), scale, threads)
    return o, lse


def attention_bwd(q, k, v, o, do, lse, causal=False, scale=None, threads=0):
    """Backward of attention: float32 [B, H, S, D] inputs, lse [B, H, S]
    (natural log, as returned by `attention`). Returns (dq, dk, dv)."""
    L = load()
    q, k, v, o, do = (np.ascontiguousarray(x, dtype=np.float32) for x in (q, k, v, o, do))
    lse = np.ascontiguousarray(lse, dtype=np.float32)
    B, H, S, D = q.shape
    scale = float(scale if scale is not None else 1.0 / np.sqrt(D))
    dq, dk, dv = (np.empty_like(q) for _ in range(3))
    L.oracle_attention_bwd(_p(q), _p(k), _p(v), _p(o), _p(do), _p(lse), _p(dq), _p(dk), _p(dv), B, H, S, D,
                           int(causal), scale, threads)
    return dq, dk, dv


def gemm_tn(a, b, threads=0):
    L = load()
    a, b = (np.ascontiguousarray(x, dtype=np.float32) for x in (a, b))
    M, K = a.shape
    N = b.shape[0]
    c = np.empty((M, N), dtype=np.float32)
    L.oracle_gemm_tn(_p(a), _p(b), _p(c), M, N, K, threads)
    return c


def round_bf16(x):
    x = np.ascontiguousarray(x, dtype=np.float32).copy()
    load().oracle_round_bf16(_p(x), x.size)
    return x


def bf16_bits(x):
    """float32 (already bf16-representable) -> uint16 bit patterns."""
    return (np.ascontiguousarray(x, dtype=np.float32).view(np.uint32) >> 16).astype(np.uint16)


def from_bf16_bits(b):
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)
