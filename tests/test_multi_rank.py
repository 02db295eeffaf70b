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

from paper_2512_18134_b200.shard import pair_range, shard_seed


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
