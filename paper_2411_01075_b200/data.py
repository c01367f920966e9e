"""Deterministic synthetic token batches.

Token (step, global sample s, position t) = splitmix64(seed, step, s, t) mod V,
computed on the host with numpy so the GPU path and the CPU oracle see the
identical batch. Rank i owns global samples [sum_{j<i} b_j, sum_{j<=i} b_j)
and its microbatch k is the k-th block of m_i of them ("each
process's data loader is configured to load its assigned batch size").
"""
from __future__ import annotations

import numpy as np

from .core import TrainPlan

_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_G = np.uint64(0x9E3779B97F4A7C15)


def _mix(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def tokens(samples: np.ndarray, seq: int, vocab: int, seed: int, step: int) -> np.ndarray:
    """int32 [len(samples), seq + 1]: inputs are [:, :-1], next-token targets [:, 1:]."""
    s = np.asarray(samples, dtype=np.uint64)[:, None]
    t = np.arange(seq + 1, dtype=np.uint64)[None, :]
    with np.errstate(over="ignore"):
        key = _mix(np.uint64(seed) * _G + np.uint64(step))
        z = _mix(key + s * np.uint64(0x100000001B3) + t * _G)
    return (z % np.uint64(vocab)).astype(np.int32)


def rank_samples(plan: TrainPlan, rank: int) -> np.ndarray:
    start = sum(a.batch for a in plan.assignments[:rank])
    return np.arange(start, start + plan.assignments[rank].batch, dtype=np.int64)


def rank_tokens(plan: TrainPlan, rank: int, seq: int, vocab: int, seed: int,
                step: int) -> np.ndarray:
    return tokens(rank_samples(plan, rank), seq, vocab, seed, step)
