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


# ---------------------------------------------------------------------------------------------
# Corrected-covariance weighting: a reported VARIANT, not the paper's Theorem 1.
#
# Theorem 1 wants w = argmin Var(sum w_i X_i) s.t. sum w_i = 1, i.e. w ∝ Cov(X)^{-1} 1,
# but its printed matrices do not follow from its own Lemmas (reading Q6; SURVEY App. A.8-A.9:
# for C1's b the printed weights have LARGER variance than uniform weights).  Here Cov(X) is the
# exact covariance under the paper's own model -- g_i = mean of b_i iid N(G, Sigma) samples,
# independent across nodes (Eq. 1), g = sum r_j g_j (Eq. 9) -- from Isserlis' theorem:
# for jointly Gaussian x, y with means mu_x, mu_y and cross-covariance C,
#     Cov(x^T x, y^T y) = 2 tr(C C^T) + 4 mu_x^T C mu_y.
# Cov(g_i, g_j) = delta_ij Sigma / b_i,  Cov(g, g_i) = r_i Sigma / b_i = Sigma / B,  Cov(g, g) = Sigma / B, so
#     Var|g_i|^2 = tau / b_i^2 + c / b_i,   Cov(|g|^2, |g_i|^2) = Var|g|^2 = tau / B^2 + c / B,
#     Cov(|g_i|^2, |g_j|^2) = 0 (i != j),   tau = 2 tr(Sigma^2),  c = 4 G^T Sigma G.
# Propagated through Eq. 10 and divided by c (a common factor does not change w), with
# rho = tau / c and k_i = b_i B / (B - b_i):
#     A_G(i,j) = [rho (1 - (b_i + b_j)/B + delta_ij) + (B - b_i - b_j + delta_ij b_i)] / ((B-b_i)(B-b_j))
#     A_S(i,j) = k_i k_j [delta_ij (rho / b_i^2 + 1 / b_i) - (rho / B^2 + 1 / B)]
# For isotropic Sigma = (trS/d) I: rho = 2 (trS)^2/d / (4 |G|^2 trS / d) = trS / (2 |G|^2)
# = B_noise / 2 -- d cancels.  rho = 0 is the first-order (delta-method) limit, whose A_S diagonal
# B b_i/(B - b_i) equals Theorem 1's printed a_S(i,i).
# ---------------------------------------------------------------------------------------------
def corrected_matrices(b, rho: float):
    """Exact Gaussian Cov of (G_i) and (S_i), divided by c = 4 G^T Sigma G (derivation above)."""
    b = [float(x) for x in b]
    n = len(b)
    B = sum(b)
    AG = np.empty((n, n))
    AS = np.empty((n, n))
    for i in range(n):
        for j in range(n):
            bi, bj = b[i], b[j]
            dij = 1.0 if i == j else 0.0
            AG[i, j] = ((rho * (1.0 - (bi + bj) / B + dij) + (B - bi - bj + dij * bi))
                        / ((B - bi) * (B - bj)))
            ki, kj = bi * B / (B - bi), bj * B / (B - bj)
            AS[i, j] = ki * kj * (dij * (rho / (bi * bi) + 1.0 / bi) - (rho / (B * B) + 1.0 / B))
    return AG, AS


RHO_MIN, RHO_MAX = 1e-12, 1e12


def gns_estimate_corrected(local_sq, global_sq: float, b, rho: float | None = None) -> dict:
    """Eq. 10 estimates combined with the corrected-covariance weights w = A^{-1} 1 / (1^T A^{-1} 1)
    (A symmetric).  rho None: rho = B_noise / 2 of the Theorem-1 estimate, clamped to
    [RHO_MIN, RHO_MAX] (B_noise <= 0 or NaN -> RHO_MAX).  (The weights turn out not to depend on
    rho at all -- w_i = (B - b_i) / ((n-1) B) for both G and S -- which the tests pin; the oracle
    still follows the general construction step by step.)  rho = 0 makes A_S singular: the
    first-order covariance of sum (B - b_i) S_i vanishes."""
    if len(b) < 2:
        raise ValueError("the heterogeneous GNS needs n >= 2 (Eq. 10 divides by B - b_i)")
    Gi, Si = local_estimates(local_sq, global_sq, b)
    if rho is None:
        t = gns_estimate(local_sq, global_sq, b)
        G0, S0 = t["G2"], t["trS"]
        rho = RHO_MAX if not (G0 > 0.0) or not (S0 == S0) else min(max(S0 / G0 / 2.0, RHO_MIN), RHO_MAX)
    AG, AS = corrected_matrices(b, float(rho))
    wG, wS = optimal_weights(AG), optimal_weights(AS)
    G = 0.0
    S = 0.0
    for i in range(len(b)):
        G += wG[i] * Gi[i]
        S += wS[i] * Si[i]
    with np.errstate(divide="ignore", invalid="ignore"):
        Bn = float(np.float64(S) / np.float64(G))
    return {"G2": G, "trS": S, "B_noise": Bn, "wG": wG, "wS": wS, "Gi": Gi, "Si": Si,
            "rho": float(rho)}
