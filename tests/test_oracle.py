"""The C oracle (oracle/attention.c, oracle/gemm.c) against independent numpy
restatements. CPU only. The attention oracle's numerics are parity-UNPINNED by
the reference (it has no attention code); these tests pin its internal
consistency: two-pass == online-softmax order, causal masking, LSE, ragged
shapes, bf16 rounding."""
import numpy as np
import pytest

from tests import oracle_lib


def np_attention(q, k, v, causal, scale):
    s = np.einsum("bhqd,bhkd->bhqk", q.astype(np.float64), k.astype(np.float64)) * scale
    if causal:
        Sq, Sk = s.shape[-2:]
        mask = np.arange(Sk)[None, :] > np.arange(Sq)[:, None]
        s = np.where(mask, -np.inf, s)
    m = s.max(-1, keepdims=True)
    p = np.exp(s - m)
    l = p.sum(-1, keepdims=True)
    o = np.einsum("bhqk,bhkd->bhqd", p / l, v.astype(np.float64))
    return o, (m + np.log(l))[..., 0]


@pytest.mark.parametrize("B,H,S,D,causal", [(1, 2, 64, 32, False), (2, 1, 100, 64, True), (1, 1, 1, 16, False),
                                            (1, 2, 129, 128, True)])
def test_two_pass_matches_numpy(B, H, S, D, causal):
    rng = np.random.default_rng(0)
    q, k, v = (rng.standard_normal((B, H, S, D), dtype=np.float32) for _ in range(3))
    o, lse = oracle_lib.attention(q, k, v, causal=causal)
    ro, rl = np_attention(q, k, v, causal, 1 / np.sqrt(D))
    assert np.abs(o - ro).max() < 1e-5
    assert np.abs(lse - rl).max() < 1e-5


@pytest.mark.parametrize("tile", [16, 128])
@pytest.mark.parametrize("causal", [False, True])
def test_online_order_matches_two_pass(tile, causal):
    rng = np.random.default_rng(1)
    q, k, v = (rng.standard_normal((1, 3, 300, 64), dtype=np.float32) for _ in range(3))
    a, la = oracle_lib.attention(q, k, v, causal=causal)
    b, lb = oracle_lib.attention(q, k, v, causal=causal, online=True, tile=tile)
    assert np.abs(a - b).max() < 1e-4
    assert np.abs(la - lb).max() < 1e-4


def test_query_prefix_against_full_keys():
    rng = np.random.default_rng(2)
    q, k, v = (rng.standard_normal((1, 1, 200, 32), dtype=np.float32) for _ in range(3))
    full, lf = oracle_lib.attention(q, k, v, causal=True)
    part, lp = oracle_lib.attention(q[:, :, :50], k, v, causal=True)
    assert np.abs(full[:, :, :50] - part).max() == 0
    assert np.abs(lf[:, :, :50] - lp).max() == 0


def test_c1_config_cpu_reference_run():
    """BASELINE config 1's host attention: B=1 H=2 S=512 d=64, seed 7,
    N(0,1) inputs rounded through bf16."""
    rng = np.random.default_rng(7)
    q, k, v = (oracle_lib.round_bf16(rng.standard_normal((1, 2, 512, 64), dtype=np.float32)) for _ in range(3))
    o, lse = oracle_lib.attention(q, k, v)
    ro, rl = np_attention(q, k, v, False, 1 / 8)
    assert np.abs(o - ro).max() < 1e-5 and np.isfinite(lse).all()


def test_gemm_matches_numpy():
    rng = np.random.default_rng(3)
    a = rng.standard_normal((70, 33), dtype=np.float32)
    b = rng.standard_normal((45, 33), dtype=np.float32)
    assert np.abs(oracle_lib.gemm_tn(a, b) - a.astype(np.float64) @ b.T.astype(np.float64)).max() < 1e-4


def test_bf16_rounding_is_round_to_nearest_even():
    x = np.array([1.0, 1.00390625, 1.005859375, -3.14159, 65504.0, 1e-30, np.inf, -np.inf], dtype=np.float32)
    r = oracle_lib.round_bf16(x)
    import torch
    t = torch.from_numpy(x).to(torch.bfloat16).float().numpy()
    assert np.array_equal(r, t)
    bits = oracle_lib.bf16_bits(r)
    assert np.array_equal(oracle_lib.from_bf16_bits(bits), r)


@pytest.mark.parametrize("causal", [False, True])
def test_backward_matches_float64_autograd(causal):
    # the backward restatement against torch autograd in float64 (CPU): an
    # independent derivation of the same gradients
    import torch
    rng = np.random.default_rng(3)
    B, H, S, D = 1, 2, 80, 32
    q, k, v, do = (rng.standard_normal((B, H, S, D)).astype(np.float32) for _ in range(4))
    o, lse = oracle_lib.attention(q, k, v, causal=causal)
    dq, dk, dv = oracle_lib.attention_bwd(q, k, v, o, do, lse, causal=causal)
    tq, tk, tv = (torch.tensor(x, dtype=torch.float64, requires_grad=True) for x in (q, k, v))
    out = torch.nn.functional.scaled_dot_product_attention(tq, tk, tv, is_causal=causal)
    out.backward(torch.tensor(do, dtype=torch.float64))
    for mine, t in ((dq, tq), (dk, tk), (dv, tv)):
        assert np.abs(mine - t.grad.numpy()).max() < 1e-5
