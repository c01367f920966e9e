"""Comparison metrics shared by the parity tests — TEST INFRASTRUCTURE ONLY.

max_rel: element-wise relative error with a floor of `floor * max|ref|` (1%)
in the denominator: elements within 100x of the tensor's largest magnitude
are judged element-wise; elements that cancel to ~0 (e.g. AdamW moments where
0.9 m + 0.1 g ~ 0, where one FMA-vs-separate rounding is a few ulps of the
operands) are judged against 1% of the tensor's scale instead of against
their own vanishing magnitude. fp32 bar (north_star): max_rel <= 1e-5.

norm_rel: ||a - b||_2 / ||b||_2, used for gradients computed from bf16
activations against an fp32 reference (north_star bar: 2e-2).
"""
from __future__ import annotations

import numpy as np

FP32_RTOL = 1e-5
BF16_GRAD_RTOL = 2e-2


def max_rel(a, b, floor: float = 1e-2) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.size == 0:
        return 0.0
    scale = float(np.max(np.abs(b)))
    den = np.maximum(np.abs(b), max(floor * scale, 1e-30))
    return float(np.max(np.abs(a - b) / den))


def norm_rel(a, b) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))
