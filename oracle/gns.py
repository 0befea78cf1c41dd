"""Oracle: heterogeneous gradient-noise-scale estimator, exactly as PAPER.md §4.4 defines it.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Eq. 10:
    G_i = (B |g|^2 - b_i |g_i|^2) / (B - b_i)
    S_i = b_i B / (B - b_i) * (|g_i|^2 - |g|^2)
Theorem 1 / Eq. 11 (restated P:769-799):
    w^G = 1^T A_G^{-1} / (1^T A_G^{-1} 1),   w^S = 1^T A_S^{-1} / (1^T A_S^{-1} 1)
    a_G(i,i) = (B + 2 b_i) / (B^2 - B b_i)
    a_G(i,j) = (B^2 - b_i^2 - b_j^2) / (B (B - b_i)(B - b_j))        i != j
    a_S(i,i) = B b_i / (B - b_i)
    a_S(i,j) = b_i b_j (B - b_i - b_j) / ((B - b_i)(B - b_j))         i != j
    G = sum_i w^G_i G_i,  S = sum_i w^S_i S_i   (rank order)
P:364:  B_noise = S / G.

The printed Theorem-1 entries are implemented verbatim (reading Q6 of DESIGN.md §4: the theorem is
internally inconsistent with App. B, but unbiasedness holds for any weights summing to 1, which
is what the pins check).  The row vector 1^T A^{-1} is obtained as solve(A^T, 1) with LAPACK gesv
(Gaussian elimination with partial pivoting) -- a library primitive used as one step.
"""
from __future__ import annotations

import numpy as np


def local_estimates(local_sq, global_sq: float, b):
    """Eq. 10 for every node i; requires 0 < b_i < B."""
    b = [float(x) for x in b]
    B = sum(b)
    Gi, Si = [], []
    for i, bi in enumerate(b):
        if not (0.0 < bi < B):
            raise ValueError("Eq. 10 needs 0 < b_i < B")
        Gi.append((B * global_sq - bi * float(local_sq[i])) / (B - bi))
        Si.append(bi * B / (B - bi) * (float(local_sq[i]) - global_sq))
    return np.array(Gi), np.array(Si)


def weight_matrices(b):
    """Theorem 1's A_G and A_S, entry by entry as printed."""
    b = [float(x) for x in b]
    n = len(b)
    B = sum(b)
    AG = np.empty((n, n))
    AS = np.empty((n, n))
    for i in range(n):
        for j in range(n):
            bi, bj = b[i], b[j]
            if i == j:
                AG[i, j] = (B + 2.0 * bi) / (B * B - B * bi)
                AS[i, j] = B * bi / (B - bi)
            else:
                AG[i, j] = (B * B - bi * bi - bj * bj) / (B * (B - bi) * (B - bj))
                AS[i, j] = bi * bj * (B - bi - bj) / ((B - bi) * (B - bj))
    return AG, AS


def optimal_weights(A) -> np.ndarray:
    """Eq. 11: w = 1^T A^{-1} / (1^T A^{-1} 1)."""
    n = A.shape[0]
    ones = np.ones(n)
    x = np.linalg.solve(A.T, ones)          # x^T = 1^T A^{-1}
    return x / float(np.sum(x))


def gns_estimate(local_sq, global_sq: float, b) -> dict:
    """Full §4.4 pipeline: Eq. 10 -> Theorem 1 weights -> G, S -> B_noise = S / G."""
    if len(b) < 2:
        raise ValueError("the heterogeneous GNS needs n >= 2 (Eq. 10 divides by B - b_i)")
    Gi, Si = local_estimates(local_sq, global_sq, b)
    AG, AS = weight_matrices(b)
    wG = optimal_weights(AG)
    wS = optimal_weights(AS)
    G = 0.0
    S = 0.0
    for i in range(len(b)):
        G += wG[i] * Gi[i]
        S += wS[i] * Si[i]
    with np.errstate(divide="ignore", invalid="ignore"):
        Bn = float(np.float64(S) / np.float64(G))
    return {"G2": G, "trS": S, "B_noise": Bn,
            "wG": wG, "wS": wS, "Gi": Gi, "Si": Si}
