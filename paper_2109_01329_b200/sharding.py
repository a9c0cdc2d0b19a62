"""Counter-offset sharding of one stream across GPUs.

The reference splits an element range across workers by giving chunk
[start, stop) the state skip_ahead(base, start) (rngburn.py:70-73,
execution.py:309-315); gaussian chunks start on a pair boundary
(rngburn.py:84-89).  The same rule places each GPU's slice: rank g generates
words [s_g, s_{g+1}) of the single stream with no collective, and
concatenating the slices reproduces the single-stream output bit for bit.
"""

from __future__ import annotations

from dataclasses import dataclass

from .distributions import DistributionSpec, Gaussian, Lognormal, generate, words_consumed
from .engine import EngineState, Mrg32k3a, Philox4x32x10, skip_ahead


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    start: int  # first element of the global request
    count: int  # elements on this rank


def strong_shard(n_total: int, rank: int, world: int, align: int = 4) -> Shard:
    """Rank's part of a fixed total: [floor_align(r*n/G), floor_align((r+1)*n/G)),
    the last rank taking the remainder.  `align` keeps slice starts on
    16-byte / pair boundaries."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")

    def edge(g):
        if g >= world:
            return n_total
        return (g * n_total // world) // align * align

    lo, hi = edge(rank), edge(rank + 1)
    return Shard(rank, world, lo, max(0, hi - lo))


def weak_shard(n_per_rank: int, rank: int, world: int) -> Shard:
    """Fixed work per rank: rank r owns elements [r*n, (r+1)*n) of the stream."""
    return Shard(rank, world, rank * n_per_rank, n_per_rank)


def shard_state(spec: DistributionSpec, base: EngineState, shard: Shard) -> EngineState:
    """Engine state at the shard's first element (pairs count 2 words per 2 samples).
    A stateful engine object is read, not advanced."""
    if isinstance(base, (Philox4x32x10, Mrg32k3a)):
        base = base.state
    if isinstance(spec, (Gaussian, Lognormal)) and shard.start % 2:
        raise ValueError("gaussian/lognormal shards must start on an even element")
    return skip_ahead(base, words_consumed(spec, shard.start) if shard.start else 0)


def generate_shard(spec: DistributionSpec, base: EngineState, shard: Shard, out=None, stream=None):
    """This rank's slice of the global request, generated locally."""
    return generate(spec, shard_state(spec, base, shard), shard.count, out, stream)[1]
