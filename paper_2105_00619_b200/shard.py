"""Batch-shard rule of the multi-GPU path.

Global batch t of a sampler call belongs to shard t % n_shards; every shard
runs the same cursor (so the SplitMix64 chain and the per-class permutations
are identical everywhere) and keeps its own batches.  optb_sbs_next_dev
implements the same rule on the device; these helpers are its host mirror
(used by the sampler wrapper for buffer sizes and by the CPU gloo tests).
"""
from __future__ import annotations


def shard_batches(n_batches: int, shard: int, n_shards: int) -> list:
    """Indices (within the call) of the batches shard `shard` produces, in order."""
    if n_shards < 1 or not 0 <= shard < n_shards:
        raise ValueError(f"bad shard {shard} of {n_shards}")
    return list(range(shard, n_batches, n_shards))


def shard_batch_count(n_batches: int, shard: int, n_shards: int) -> int:
    return (n_batches - shard + n_shards - 1) // n_shards if n_batches > shard else 0


def interleave(parts: list, batch: int) -> list:
    """Reassemble the global stream from per-shard outputs (flat lists of
    class-major draws, batch after batch)."""
    n_shards = len(parts)
    counts = [len(p) // batch for p in parts]
    out = []
    for t in range(sum(counts)):
        s, j = t % n_shards, t // n_shards
        out.extend(parts[s][j * batch:(j + 1) * batch])
    return out
