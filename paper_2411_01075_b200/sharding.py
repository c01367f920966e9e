"""Per-unit contiguous shard vectors: the source of truth for the uneven
flat-parameter layout on the GPUs.

Behaviour follows the reference's `assign_unit_shards`
(`pkg/src/hetplan/sharding.py:48-98`) exactly, because the offsets it emits
are the byte layout every rank's HBM buffers are built from and they must be
bit-identical to the planner's:

* walk units in order; a unit is sharded evenly (U/N each, remainder to the
  rank with the largest unmet budget, ties to the lower rank) whenever every
  rank's remaining budget still covers U/N within one parameter
  (sharding.py:71-74);
* otherwise the unit absorbs each rank's surplus over what an all-even tail
  would need, clipped to [0, U] (sharding.py:75-84; note the reference never
  rescales by the computed sum, Appendix B of SURVEY.md);
* integer rounding: truncate, clip negatives, trim an overshoot from the
  largest counts (lowest index first), then hand out the remainder one
  parameter at a time by largest credit (sharding.py:18-40);
* a vector is "even" if no entry is a full parameter away from U/N
  (sharding.py:43-45); offsets are prefix sums in rank order (89-95).
"""
from __future__ import annotations

from .core import InputError, ModelSpec, UnitShardPlan

RATIO_SUM_TOL = 1e-9
EVEN_SLACK = 1.0


def _integerise(target: list[float], total: int, unmet: list[float]) -> list[int]:
    n = len(target)
    counts = [max(int(t), 0) for t in target]
    left = total - sum(counts)
    if left < 0:
        for i in sorted(range(n), key=lambda r: (-counts[r], r)):
            cut = min(counts[i], -left)
            counts[i] -= cut
            left += cut
            if left == 0:
                break
    credit = [unmet[i] - counts[i] for i in range(n)]
    while left > 0:
        pick = 0
        for i in range(1, n):
            if credit[i] > credit[pick]:
                pick = i
        counts[pick] += 1
        credit[pick] -= 1
        left -= 1
    return counts


def _even(vec: list[int], unit_params: int, n: int) -> bool:
    share = unit_params / n
    return all(abs(v - share) < EVEN_SLACK for v in vec)


def assign_unit_shards(ratios: list[float], model: ModelSpec) -> UnitShardPlan:
    n = len(ratios)
    if n < 1:
        raise InputError("need at least one ratio")
    if any(r < 0 for r in ratios):
        raise InputError("ratios must be >= 0")
    if abs(sum(ratios) - 1.0) > RATIO_SUM_TOL:
        raise InputError(f"ratios sum to {sum(ratios)!r}, expected 1")

    L, U = model.layers, model.params_per_layer
    left = [r * model.total_params for r in ratios]
    shard_rows: list[tuple[int, ...]] = []
    offset_rows: list[tuple[int, ...]] = []
    n_uneven = 0
    for u in range(L):
        share = U / n
        if all(left[i] - share >= -EVEN_SLACK for i in range(n)):
            vec = _integerise([share] * n, U, left)
        else:
            tail = (L - u - 1) * U / n
            want = [min(max(left[i] - tail, 0.0), float(U)) for i in range(n)]
            if sum(want) <= 0:
                want = [share] * n
            vec = _integerise(want, U, left)
        if not _even(vec, U, n):
            n_uneven += 1
        starts = []
        pos = 0
        for i in range(n):
            left[i] -= vec[i]
            starts.append(pos)
            pos += vec[i]
        shard_rows.append(tuple(vec))
        offset_rows.append(tuple(starts))
    return UnitShardPlan(units=L, uneven_units=n_uneven,
                         shards=tuple(shard_rows), offsets=tuple(offset_rows))
