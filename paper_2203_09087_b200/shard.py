"""Multi-GPU z-slab sharding: one process per GPU.

Each rank owns a contiguous range of axis-0 planes (a balanced floor/ceil
split -- the reference's even_plan, streaming.hpp:50-58, may return fewer
ranges than ranks) plus one halo plane per side where the image has one
(chunk.hpp:193-220 semantics).  A rank accumulates its slab's int64
histogram (change sums + voxel counts per bin) on its GPU; the ONLY exchange
is one all_reduce(sum) of that histogram, after which every rank runs K3.
The result is bit-identical for every rank count because the histogram is
an integer sum (the reference's chunk invariance, acceptance.cpp:203-227).

The functions take the accumulate / finalize steps as callables so the same
driver runs over NCCL on GPUs (bench.py) and over gloo on CPU in the tests,
where the oracle plays the per-slab accumulate (tests/test_multigpu_gloo.py).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable


@dataclass(frozen=True)
class Shard:
    rank: int
    own0: int      # first owned plane
    own1: int      # one past the last owned plane
    plane0: int    # first plane held (own0 - 1 when a halo plane exists)
    plane1: int    # one past the last plane held

    @property
    def planes(self) -> int:
        return self.plane1 - self.plane0


def shard_bounds(w0: int, world: int, rank: int) -> Shard:
    """Rank `rank`'s share of [0, w0): sizes differ by at most one plane,
    every rank gets at least one plane when w0 >= world, and a rank beyond
    w0 owns nothing (own0 == own1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    base, extra = divmod(w0, world)
    own0 = rank * base + min(rank, extra)
    own1 = own0 + base + (1 if rank < extra else 0)
    return Shard(rank, own0, own1, max(own0 - 1, 0) if own1 > own0 else own0,
                 min(own1 + 1, w0) if own1 > own0 else own0)


def sharded_histogram(shard: Shard, accumulate: Callable, hist, all_reduce: Callable):
    """accumulate(shard, hist) adds this rank's slab into `hist` (zeroed by
    the caller); all_reduce(hist) sums it across ranks in place."""
    if shard.own1 > shard.own0:
        accumulate(shard, hist)
    all_reduce(hist)
    return hist
