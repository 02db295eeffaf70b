"""B x H sharding of an FA-forward job over the GPUs of one box.

Every (batch, head) pair is an independent attention problem, so the job is
split into contiguous ranges of the flattened B*H pairs, one per rank, with
no collective on the data path. Each rank generates and owns
only its own pairs and runs the same plan on them. The only collectives are
outside the timed region: the start/stop barriers, the max-over-ranks of the
elapsed time, and the gather of per-pair checksums / clock summaries.

The inputs of pair p are generated from a generator seeded with
pair_seed(seed, p), so the job's data, and therefore its output, does not
depend on how many ranks share it: the per-pair checksums of a run on N GPUs
equal those of the same job on one GPU (tests/test_multi_rank.py checks this
with two gloo ranks, bench.py reports the job checksum).
"""
import hashlib


def pair_range(num_pairs, world, rank):
    """[start, stop) of the flattened (b, h) pairs owned by `rank`: the first
    num_pairs % world ranks get one extra pair."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(num_pairs, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def shard_seed(seed, rank):
    """Per-shard generator seed (BASELINE s8d: seed + shard index)."""
    return seed + rank


def pair_seed(seed, pair):
    """Generator seed of one (b, h) pair: independent of the sharding."""
    return (seed << 20) + pair


class PairShard:
    """The pairs [start, stop) of a B*H-pair job owned by one rank."""

    def __init__(self, num_pairs, world, rank):
        self.num_pairs = num_pairs
        self.world = world
        self.rank = rank
        self.start, self.stop = pair_range(num_pairs, world, rank)

    @property
    def count(self):
        return self.stop - self.start

    def make_inputs(self, S, D, seed, device, dtype):
        """q, k, v of this shard as [1, count, S, D] tensors (the flattened
        pairs are the kernel's B*H axis); pair p drawn from N(0, 1) with its
        own generator, so the values do not depend on the sharding."""
        import torch
        n = max(self.count, 0)
        q, k, v = (torch.empty((1, n, S, D), device=device, dtype=dtype) for _ in range(3))
        g = torch.Generator(device=device)
        for i in range(n):
            g.manual_seed(pair_seed(seed, self.start + i))
            x = torch.randn((3, S, D), device=device, generator=g)
            q[0, i].copy_(x[0])
            k[0, i].copy_(x[1])
            v[0, i].copy_(x[2])
        return q, k, v

    def checksums(self, o, chunk=64):
        """Per-pair exact checksum of a [1, count, S, D] bf16 / fp16 output:
        the int64 sum of its 16-bit patterns (order-independent, so identical
        for any sharding and any reduction order)."""
        import torch
        x = o.reshape(o.shape[1], -1).view(torch.int16)
        out = torch.empty(x.shape[0], dtype=torch.int64, device=o.device)
        for a in range(0, x.shape[0], chunk):
            out[a:a + chunk] = x[a:a + chunk].to(torch.int64).sum(dim=1)
        return out


def gather_pair_checksums(local, shard, dist=None):
    """All per-pair checksums of the job (on every rank), in pair order.
    `local` is this rank's [count] int64 tensor; shards may differ in size."""
    import torch
    if shard.world == 1 or dist is None:
        return local.cpu()
    mx = -(-shard.num_pairs // shard.world)
    pad = torch.zeros(mx, dtype=torch.int64, device=local.device)
    pad[: local.numel()] = local
    out = [torch.zeros_like(pad) for _ in range(shard.world)]
    dist.all_gather(out, pad)
    parts = []
    for r in range(shard.world):
        a, b = pair_range(shard.num_pairs, shard.world, r)
        parts.append(out[r][: b - a].cpu())
    return torch.cat(parts)


def job_digest(pair_checksums):
    """Short digest of the whole job's output (all pairs, in order)."""
    import numpy as np
    arr = np.asarray(pair_checksums, dtype=np.int64)
    return hashlib.sha256(arr.tobytes()).hexdigest()[:16]
