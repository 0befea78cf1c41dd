"""Oracle: weighted gradient aggregation (Eq. 9) and the squared norms feeding Eq. 10.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md:326-331 (§4.3, Eq. 9):   g = sum_{i in N} r_i g_i,   r_i = b_i / B  (§3.1)
PAPER.md:125-130 (§2.1, Eq. 1):   g_i is node i's *mean* local gradient over its b_i samples.
PAPER.md:339-343 (§4.4, Eq. 10):  the estimators need |g_i|^2 and |g|^2.

Arithmetic is float64, ranks summed in ascending order, no FMA (numpy never contracts).  The
inputs of record are the fp32 values or bf16 bit patterns produced by ``cannikin_synth``; they are
up-converted exactly to float64 here.
"""
from __future__ import annotations

import math

import numpy as np


def to_f64(x: np.ndarray, dtype: str) -> np.ndarray:
    """Exact up-conversion of an input of record to float64.

    bf16 bits: a bfloat16 is the top 16 bits of an IEEE float32, so shifting left by 16 gives the
    float32 with the same value, which converts exactly to float64.
    """
    if dtype == "f32":
        return np.asarray(x, dtype=np.float32).astype(np.float64)
    if dtype == "bf16":
        u32 = np.asarray(x, dtype=np.uint16).astype(np.uint32) << np.uint32(16)
        return u32.view(np.float32).astype(np.float64)
    raise ValueError(dtype)


def ratios(b) -> np.ndarray:
    """r_i = b_i / B with B = sum_i b_i."""
    b = np.asarray(b, dtype=np.float64)
    B = float(np.sum(b))
    return np.array([bi / B for bi in b], dtype=np.float64)


def weighted_sum(gs64, r) -> np.ndarray:
    """Eq. 9: g = sum_i r_i g_i, accumulated in float64 in fixed rank order i = 0..n-1 (O-2)."""
    n = len(gs64)
    assert n == len(r) and n >= 1
    acc = np.zeros_like(np.asarray(gs64[0], dtype=np.float64))
    for i in range(n):
        acc = acc + float(r[i]) * np.asarray(gs64[i], dtype=np.float64)
    return acc


def sq_norm(x64) -> float:
    """|x|^2 = sum_e x_e^2 in float64 (pairwise summation by numpy's add.reduce; O-3)."""
    x = np.asarray(x64, dtype=np.float64)
    return float(np.add.reduce(x * x)) if x.size else 0.0


def sq_norm_exact(x64) -> float:
    """|x|^2 with a correctly-rounded sum of the float64 squares (math.fsum) -- small N only."""
    x = np.asarray(x64, dtype=np.float64)
    return math.fsum((x * x).tolist())


def aggregate(gs, r, dtype: str):
    """The whole single-pass contract of the hot path on host inputs of record.

    Returns (g, local_sq[n], global_sq) with g = Eq. 9 in float64, local_sq[i] = |g_i|^2,
    global_sq = |g|^2 of the exact-double aggregate (reading Q2 of DESIGN.md §4).
    """
    gs64 = [to_f64(g, dtype) for g in gs]
    g = weighted_sum(gs64, r)
    local_sq = np.array([sq_norm(x) for x in gs64])
    return g, local_sq, sq_norm(g)


def elementwise_scale(gs64, r) -> np.ndarray:
    """sum_i |r_i g_i[e]| per element: the magnitude scale of the cancellation-aware error metric
    (reading Q1 of DESIGN.md §4): err_e = |gpu_e - ref_e| / max(sum_i |r_i g_i[e]|, 1e-30)."""
    acc = np.zeros_like(np.asarray(gs64[0], dtype=np.float64))
    for i in range(len(gs64)):
        acc = acc + np.abs(float(r[i]) * np.asarray(gs64[i], dtype=np.float64))
    return acc
