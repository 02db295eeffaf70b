"""Multi-GPU driver logic on CPU: world_size-2 gloo process groups stand in for
two B200s. The B x H sharding must cover every (b, h) pair exactly once, and
stitching the per-rank results must reproduce the single-process answer (the
oracle plays the kernel here; the shard logic is what is under test)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2512_18134_b200.shard import PairShard, job_digest, pair_range, shard_seed


def test_pair_ranges_partition():
    for P in (1, 7, 128, 1024):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                a, b = pair_range(P, world, r)
                seen.extend(range(a, b))
            assert seen == list(range(P))
    with pytest.raises(ValueError):
        pair_range(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from tests import oracle_lib
    B, H, S, D = 2, 3, 64, 16
    rng = np.random.default_rng(5)
    qkv = rng.standard_normal((3, B * H, S, D), dtype=np.float32)
    a, b = pair_range(B * H, world, rank)
    o, lse = oracle_lib.attention(qkv[0, a:b][None], qkv[1, a:b][None], qkv[2, a:b][None], causal=True)
    # gather variable-size shards (pad to the largest)
    n = torch.tensor([b - a])
    sizes = [torch.zeros(1, dtype=torch.long) for _ in range(world)]
    dist.all_gather(sizes, n)
    mx = int(max(s.item() for s in sizes))
    pad = torch.zeros((mx, S, D))
    pad[: b - a] = torch.from_numpy(o[0])
    out = [torch.zeros_like(pad) for _ in range(world)]
    dist.all_gather(out, pad)
    # elapsed-time reduction used by bench.py (max over ranks)
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        full = torch.cat([out[r][: int(sizes[r].item())] for r in range(world)]).numpy()
        ref, _ = oracle_lib.attention(qkv[0][None], qkv[1][None], qkv[2][None], causal=True)
        q.put((float(np.abs(full - ref[0]).max()), t.item(), [shard_seed(2026, r) for r in range(world)]))
    dist.destroy_process_group()


def test_two_rank_gloo_sharded_job_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    err, tmax, seeds = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert err == 0.0
    assert tmax == 2.0
    assert seeds == [2026, 2027]


def _mock_fa(q, k, v):
    """Stand-in for the CUDA kernel on CPU: the fp32 oracle on the bf16
    inputs, rounded to bf16 (the shard logic is what is under test)."""
    from tests import oracle_lib
    o, _ = oracle_lib.attention(q.float().numpy(), k.float().numpy(), v.float().numpy())
    return torch.from_numpy(o).to(torch.bfloat16)


def _bench_worker(rank, world, port, q, job_pairs, S, Dh):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(world), RANK=str(rank),
                      LOCAL_RANK=str(rank))
    import bench
    ranks = bench.Ranks(device="cpu")
    shard = PairShard(job_pairs, world, rank)
    qq, kk, vv = shard.make_inputs(S, Dh, 3008, "cpu", torch.bfloat16)
    o = _mock_fa(qq, kk, vv)
    cks = ranks.gather_checksums(shard.checksums(o), shard)
    t = ranks.max(float(rank + 1))
    per_rank = ranks.gather_objects({"rank": rank, "pairs": [shard.start, shard.stop]})
    ranks.barrier()
    if rank == 0:
        q.put((cks.tolist(), job_digest(cks.numpy()), t, per_rank))
    ranks.close()


@pytest.mark.parametrize("world,job_pairs", [(2, 6), (3, 7)])
def test_bench_sharded_job_checksums_match_single_process(world, job_pairs):
    """bench.py's own path on gloo ranks (PairShard inputs, per-pair exact
    checksums, gather, digest, max-over-ranks) reproduces the one-process job."""
    S, Dh = 64, 16
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_worker, args=(r, world, port, q, job_pairs, S, Dh)) for r in range(world)]
    for p in procs:
        p.start()
    cks, digest, tmax, per_rank = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    one = PairShard(job_pairs, 1, 0)
    o1 = _mock_fa(*one.make_inputs(S, Dh, 3008, "cpu", torch.bfloat16))
    ref = one.checksums(o1)
    assert cks == ref.tolist()
    assert digest == job_digest(ref.numpy())
    assert tmax == float(world)
    assert [r["pairs"] for r in per_rank] == [list(pair_range(job_pairs, world, r)) for r in range(world)]


def test_pair_inputs_do_not_depend_on_sharding():
    full = PairShard(5, 1, 0).make_inputs(32, 16, 7, "cpu", torch.bfloat16)
    for world in (2, 5):
        for r in range(world):
            sh = PairShard(5, world, r)
            part = sh.make_inputs(32, 16, 7, "cpu", torch.bfloat16)
            for a, b in zip(part, full):
                assert torch.equal(a[0], b[0, sh.start:sh.stop])


def test_checksum_is_exact_and_order_independent():
    sh = PairShard(3, 1, 0)
    o = torch.randn(1, 3, 40, 16).to(torch.bfloat16)
    c = sh.checksums(o, chunk=2)
    bits = o.view(torch.int16).to(torch.int64)
    assert c.tolist() == [int(bits[0, i].sum()) for i in range(3)]
    o2 = o.clone()
    o2[0, 1, 5, 3] = -o2[0, 1, 5, 3] if o2[0, 1, 5, 3] != 0 else 1.0
    assert sh.checksums(o2).tolist()[1] != c.tolist()[1]


def test_self_launch_command(monkeypatch):
    """`bench.py --gpus N` outside torchrun re-launches itself with one
    process per GPU (torch.distributed.run, 127.0.0.1, NCCL_DEBUG=INFO)."""
    import bench
    seen = {}

    def fake_call(cmd, env):
        seen["cmd"], seen["env"] = cmd, env
        return 0

    monkeypatch.setattr(bench.subprocess, "call", fake_call)
    monkeypatch.setattr(bench.sys, "argv", ["bench.py", "--gpus", "4", "--steps", "3", "--share-gpu"])
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    assert bench.main() == 0
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd
    assert cmd[-5:] == ["--gpus", "4", "--steps", "3", "--share-gpu"]
    assert seen["env"]["NCCL_DEBUG"] in ("INFO", os.environ.get("NCCL_DEBUG"))
