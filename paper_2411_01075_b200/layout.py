"""Per-rank uneven flat-shard layout in HBM, derived from the planner's
UnitShardPlan (reference core.py:229-240; offsets from sharding.py:89-95).

Logical layout (bit-exact with the plan): unit u's flat vector of U params
is split into contiguous ranges [offsets[u][j], offsets[u][j] + shards[u][j])
owned by rank j. Ranks own whole ranges, never strided pieces.

Physical layout on rank i: one flat fp32 buffer per state tensor (master
param, reduced grad, AdamW m and v) plus a bf16 shadow of the master (the
all-gather send buffer), each the concatenation over units of rank i's
ranges. Every unit's local range starts on a 64-element (256 B) boundary so
all kernels get 16-byte-aligned vectors even when a shard has an odd length
(e.g. GPT-2 small at r=683/1024 owns 3,571,623 params of its last unit —
SURVEY.md §7 "Misaligned shards"); the pads are zero and stay zero under
AdamW (zero grad, zero moments). Units are indexed 0..L-1 for the
transformer blocks and L for the root unit (embeddings, final norm, tied
head), which is sharded by the same state ratios.
"""
from __future__ import annotations

from dataclasses import dataclass

from .core import InputError, ModelSpec, TrainPlan, UnitShardPlan
from .sharding import assign_unit_shards

ALIGN = 64


def _pad(n: int) -> int:
    return (n + ALIGN - 1) // ALIGN * ALIGN


@dataclass(frozen=True)
class RankLayout:
    rank: int
    nranks: int
    unit_params: int
    root_params: int
    counts: tuple[tuple[int, ...], ...]    # [L + 1][N]
    offsets: tuple[tuple[int, ...], ...]   # [L + 1][N]
    local_off: tuple[int, ...]             # [L + 1] start of rank's range in its flat buffer
    local_len: int                         # padded length of the flat buffers

    @property
    def blocks(self) -> int:
        return len(self.counts) - 1

    @property
    def root(self) -> int:
        return self.blocks

    def unit_size(self, u: int) -> int:
        return self.root_params if u == self.root else self.unit_params

    def local_range(self, u: int) -> tuple[int, int]:
        return self.local_off[u], self.counts[u][self.rank]

    def is_even(self, u: int) -> bool:
        c = self.counts[u]
        return all(x == c[0] for x in c)

    @property
    def owned_params(self) -> int:
        return sum(c[self.rank] for c in self.counts)

    @classmethod
    def build(cls, unit_shards: UnitShardPlan, root_shards: UnitShardPlan, unit_params: int,
              root_params: int, rank: int) -> "RankLayout":
        n = len(unit_shards.shards[0]) if unit_shards.units else len(root_shards.shards[0])
        if not (0 <= rank < n):
            raise InputError(f"rank {rank} outside 0..{n - 1}")
        counts = tuple(tuple(int(x) for x in row) for row in unit_shards.shards) + \
            (tuple(int(x) for x in root_shards.shards[0]),)
        offsets = tuple(tuple(int(x) for x in row) for row in unit_shards.offsets) + \
            (tuple(int(x) for x in root_shards.offsets[0]),)
        for u, (c, o) in enumerate(zip(counts, offsets)):
            size = root_params if u == len(counts) - 1 else unit_params
            if len(c) != n or sum(c) != size:
                raise InputError(f"unit {u}: shard vector does not cover {size} params")
            pos = 0
            for cj, oj in zip(c, o):
                if oj != pos or cj < 0:
                    raise InputError(f"unit {u}: offsets are not contiguous prefix sums")
                pos += cj
        local, pos = [], 0
        for c in counts:
            local.append(pos)
            pos += _pad(c[rank])
        return cls(rank=rank, nranks=n, unit_params=unit_params, root_params=root_params,
                   counts=counts, offsets=offsets, local_off=tuple(local),
                   local_len=max(pos, ALIGN))

    @classmethod
    def from_plan(cls, plan: TrainPlan, unit_params: int, root_params: int,
                  rank: int) -> "RankLayout":
        if plan.unit_shards is None:
            raise InputError("plan carries no unit_shards")
        return cls.build(plan.unit_shards, root_shard_plan(plan, root_params), unit_params,
                         root_params, rank)


def root_shard_plan(plan: TrainPlan, root_params: int) -> UnitShardPlan:
    """The root unit follows the same rule as the blocks: one unit of
    `root_params`, sharded by the plan's state ratios."""
    ratios = [a.state_ratio for a in plan.assignments]
    return assign_unit_shards(ratios, ModelSpec(layers=1, params_per_layer=root_params,
                                                global_batch=1))
