"""Shared parity check for large GPU outputs: EVERY element against the oracle, chunk by chunk.

The CUDA results and inputs of record stay on the device; each chunk of every input is copied to
the host, up-converted exactly (oracle.aggregate.to_f64), reduced by the oracle's Eq. 9
(oracle.aggregate.weighted_sum, rank order, float64) and compared with the same chunk of the
output under the Q1 metric:
    err_e = |gpu_e - ref_e| / max(sum_i |r_i g_i[e]|, 1e-30)
The oracle's norms (O-3) are accumulated over the same chunks, so a single pass yields the
element-wise maximum error and the whole-vector |g_i|^2, |g|^2 the statistics are checked against.
No arithmetic of the method lives here: only the oracle's functions and comparisons.
"""
from __future__ import annotations

import numpy as np
import torch

from oracle import aggregate as agg


def host_bits(t: torch.Tensor, dtype: str) -> np.ndarray:
    """Inputs/outputs of record as the oracle reads them (fp32 values or bf16 bit patterns)."""
    if dtype == "bf16":
        return t.view(torch.int16).cpu().numpy().view(np.uint16)
    return t.cpu().numpy()


def compare_full(outs, ins, r, dtype: str, tol: float, chunk: int = 8_000_000):
    """outs: list of device tensors that must all equal the oracle's Eq. 9 of `ins` (device
    tensors, inputs of record) with shares r.  outs[1:] must be bitwise equal to outs[0].
    Returns (max_err, local_sq[n], global_sq) with the oracle's norms over the whole vectors."""
    n = len(ins)
    N = ins[0].numel()
    lsum = np.zeros(n)
    gsum = 0.0
    max_err = 0.0
    for a in range(0, N, chunk):
        c = min(chunk, N - a)
        parts = [agg.to_f64(host_bits(g[a:a + c], dtype), dtype) for g in ins]
        ref = agg.weighted_sum(parts, r)
        scale = np.maximum(agg.elementwise_scale(parts, r), 1e-30)
        o0 = host_bits(outs[0][a:a + c], dtype)
        err = float(np.max(np.abs(agg.to_f64(o0, dtype) - ref) / scale)) if c else 0.0
        assert err <= tol, (a, err)
        max_err = max(max_err, err)
        for k in range(1, len(outs)):
            assert np.array_equal(host_bits(outs[k][a:a + c], dtype), o0), (k, a)
        for j in range(n):
            lsum[j] += agg.sq_norm(parts[j])
        gsum += agg.sq_norm(ref)
    return max_err, lsum, gsum
