"""GEMM mainloop (BASELINE config 2) parity: the Twill-scheduled TMA + tcgen05
kernel against the fp32 CPU oracle (small) and torch.matmul (full size).
Tolerance: bf16 output of an fp32-accumulated dot product -> relative 1e-2 of
the output scale."""
import numpy as np
import pytest
import torch

from tests import oracle_lib

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def plan(twfa):
    return twfa.Plan(*twfa.load_schedule("gemm_mainloop"))


# one CTA pair per 256 x 256 tile: fewer tiles than pairs, several tiles per
# pair (both TMEM accumulators, the staging double buffer), a ragged raster group
@pytest.mark.parametrize("M,N,K", [(256, 256, 64), (256, 512, 192), (512, 256, 1024), (1024, 1024, 512),
                                   (2560, 4608, 256)])
def test_gemm_matches_oracle(twfa, plan, M, N, K):
    g = torch.Generator(device="cpu").manual_seed(1234)
    a = (torch.randn(M, K, generator=g) / K ** 0.5).to(torch.bfloat16)
    b = torch.randn(N, K, generator=g).to(torch.bfloat16)
    c = twfa.gemm(plan, a.cuda(), b.cuda())
    torch.cuda.synchronize()
    ref = oracle_lib.gemm_tn(a.float().numpy(), b.float().numpy())
    err = np.abs(c.float().cpu().numpy() - ref)
    assert err.max() <= 1e-2 * max(1.0, np.abs(ref).max()), err.max()


def test_gemm_full_size(twfa, plan):
    M = N = K = 8192
    g = torch.Generator(device="cuda").manual_seed(1234)
    a = (torch.randn(M, K, device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
    b = torch.randn(N, K, device="cuda", generator=g).to(torch.bfloat16)
    c = twfa.gemm(plan, a, b)
    ref = a @ b.t()
    d = (c.float() - ref.float()).abs()
    assert d.max().item() <= 3e-2 and d.mean().item() <= 2e-3


def test_gemm_raster_groups_agree(twfa, plan, monkeypatch):
    """The raster group only reorders tiles: bit-identical C for every group."""
    g = torch.Generator(device="cuda").manual_seed(5)
    a = (torch.randn(2048, 512, device="cuda", generator=g) / 512 ** 0.5).to(torch.bfloat16)
    b = torch.randn(3072, 512, device="cuda", generator=g).to(torch.bfloat16)
    outs = []
    for grp in ("1", "3", "8", "64"):
        monkeypatch.setenv("TWFA_GEMM_GROUP", grp)
        outs.append(twfa.gemm(plan, a, b))
    for o in outs[1:]:
        assert torch.equal(o, outs[0])


@pytest.mark.parametrize("M,N,K", [(100, 256, 64), (128, 256, 64), (256, 384, 64), (256, 256, 48)])
def test_gemm_rejects_unaligned_shapes(twfa, plan, M, N, K):
    a = torch.zeros(M, K, device="cuda", dtype=torch.bfloat16)
    b = torch.zeros(N, K, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(ValueError):
        twfa.gemm(plan, a, b)


@pytest.mark.parametrize("seed", range(10))
def test_gemm_random_shapes(twfa, plan, seed):
    """Seeded fuzz over the aligned shape space (M, N multiples of 256, K of
    64) against torch's fp32 product of the same bf16 inputs: tile counts
    below, at and above the number of CTA pairs, tall and wide grids."""
    rng = np.random.default_rng(500 + seed)
    M, N = 256 * int(rng.integers(1, 17)), 256 * int(rng.integers(1, 17))
    K = 64 * int(rng.integers(1, 49))
    g = torch.Generator(device="cuda").manual_seed(600 + seed)
    a = (torch.randn(M, K, device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
    b = torch.randn(N, K, device="cuda", generator=g).to(torch.bfloat16)
    c = twfa.gemm(plan, a, b)
    ref = a.float() @ b.float().t()
    err = (c.float() - ref).abs().max().item()
    assert err <= 1e-2 * max(1.0, ref.abs().max().item()), (M, N, K, err)
