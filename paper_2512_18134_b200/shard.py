"""B x H sharding of an FA-forward job over the GPUs of one box.

Every (batch, head) pair is an independent attention problem, so the job is
split into contiguous ranges of the flattened B*H pairs, one per rank, with
no collective on the data path. Each rank generates / owns
only its own pairs and runs the same plan on them.
"""


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
