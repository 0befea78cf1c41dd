"""Pins for oracle/gns.py (Eq. 10, Theorem 1, B_noise) against hand values, closed forms and Monte Carlo."""
import math

import numpy as np
import pytest

from oracle import aggregate as agg
from oracle import gns


def test_local_estimates_spec_hand_values(golden):
    ex = golden["local_estimates"]
    b = [ex["b_i"], ex["B"] - ex["b_i"]]
    Gi, Si = gns.local_estimates([ex["local_sq"], 0.0], ex["global_sq"], b)
    assert math.isclose(Gi[0], ex["G_i"], rel_tol=1e-15)
    assert math.isclose(Si[0], ex["S_i"], rel_tol=1e-15)


def test_weight_matrix_spec_hand_values(golden):
    ex = golden["weight_matrices"]
    AG, AS = gns.weight_matrices(ex["b"])
    assert math.isclose(AG[0, 0], ex["aG00"], rel_tol=1e-15)
    assert math.isclose(AG[0, 1], ex["aG01"], rel_tol=1e-15)
    assert math.isclose(AS[0, 0], ex["aS00"], rel_tol=1e-15)
    assert AS[0, 1] == ex["aS01"]


def test_weight_matrices_symmetric_and_scale():
    """Entries scale: (b, B) -> (c b, c B) scales A_G by 1/c and A_S by c."""
    b = np.array([32.0, 64.0, 96.0])
    AG, AS = gns.weight_matrices(b)
    AG2, AS2 = gns.weight_matrices(3 * b)
    assert np.allclose(AG, AG.T, rtol=0, atol=0)
    assert np.allclose(AS, AS.T, rtol=0, atol=0)
    assert np.allclose(AG2, AG / 3, rtol=1e-14)
    assert np.allclose(AS2, AS * 3, rtol=1e-14)


@pytest.mark.parametrize("b", [[25, 75], [10, 90], [33, 41]])
def test_two_node_closed_form_weights(b):
    """n = 2 closed forms derived by hand from Theorem 1 with B = b0 + b1:
    A_G = [[(B+2b0)/(B b1), 2/B], [2/B, (B+2b1)/(B b0)]]  =>  w^G ∝ ((3b1-b0)/b0, (3b0-b1)/b1)
    A_S = diag(B b0/b1, B b1/b0)                         =>  w^S ∝ (b1^2, b0^2)."""
    b0, b1 = b
    wg = np.array([(3 * b1 - b0) / b0, (3 * b0 - b1) / b1])
    ws = np.array([b1 * b1, b0 * b0], dtype=float)
    wg /= wg.sum()
    ws /= ws.sum()
    AG, AS = gns.weight_matrices(b)
    assert np.allclose(gns.optimal_weights(AG), wg, rtol=1e-12, atol=1e-14)
    assert np.allclose(gns.optimal_weights(AS), ws, rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("n,bi", [(2, 50), (4, 16), (8, 7)])
def test_homogeneous_weights_uniform(n, bi):
    """equal b_i => exactly uniform weights (symmetry of A)."""
    AG, AS = gns.weight_matrices([bi] * n)
    assert np.allclose(gns.optimal_weights(AG), 1.0 / n, atol=1e-14)
    assert np.allclose(gns.optimal_weights(AS), 1.0 / n, atol=1e-14)


def test_weights_scale_invariant_and_sum_to_one():
    rng = np.random.default_rng(0)
    for _ in range(50):
        n = int(rng.integers(2, 9))
        b = rng.integers(1, 200, size=n).astype(float)
        wg = gns.optimal_weights(gns.weight_matrices(b)[0])
        wg5 = gns.optimal_weights(gns.weight_matrices(5 * b)[0])
        assert abs(wg.sum() - 1.0) < 1e-12
        assert np.allclose(wg, wg5, rtol=1e-9, atol=1e-12)


def test_zero_noise_gives_zero_S():
    """noiseless gradients -> S = 0, B_noise = 0, G = |G|^2."""
    b = [32, 64, 96]
    r = gns.gns_estimate([1.7, 1.7, 1.7], 1.7, b)
    assert abs(r["trS"]) < 1e-12 and abs(r["B_noise"]) < 1e-12
    assert math.isclose(r["G2"], 1.7, rel_tol=1e-12)


def test_domain_errors():
    with pytest.raises(ValueError):
        gns.gns_estimate([1.0], 1.0, [5])
    with pytest.raises(ValueError):
        gns.local_estimates([1.0, 1.0], 1.0, [0, 5])


@pytest.mark.parametrize("b", [[32, 64, 96], [25, 75], [5, 20, 40, 7]])
def test_unbiased_monte_carlo(b):
    """North-star check 2 / P:343: on Gaussian gradients with known |G|^2 and tr(Sigma), the
    Theorem-1 aggregate has E[G] = |G|^2 and E[S] = tr(Sigma): within 4 empirical standard errors.
    Per-node means are drawn exactly as the mean of b_i samples of N(G, (trS/d) I) (Eq. 1)."""
    d, trials, G2, trS = 256, 6000, 1.0, 100.0
    rng = np.random.default_rng(1234 + len(b))
    z = rng.standard_normal(d)
    G = z * np.sqrt(G2 / (z @ z))
    B = sum(b)
    r = agg.ratios(b)
    Gs, Ss = [], []
    for _ in range(trials):
        gi = [G + np.sqrt(trS / (d * bi)) * rng.standard_normal(d) for bi in b]
        g = agg.weighted_sum(gi, r)
        est = gns.gns_estimate([agg.sq_norm(x) for x in gi], agg.sq_norm(g), b)
        Gs.append(est["G2"])
        Ss.append(est["trS"])
    Gs, Ss = np.array(Gs), np.array(Ss)
    seG = Gs.std(ddof=1) / np.sqrt(trials)
    seS = Ss.std(ddof=1) / np.sqrt(trials)
    assert abs(Gs.mean() - G2) < 4 * seG, (Gs.mean(), seG)
    assert abs(Ss.mean() - trS) < 4 * seS, (Ss.mean(), seS)
    # a dropped term would bias by O(trS/B) -- far outside the band:
    assert 4 * seG < 0.25 * trS / B


def test_noise_scale_ratio():
    b = [32, 64, 96]
    r = gns.gns_estimate([1.0 + 100 / 32, 1.0 + 100 / 64, 1.0 + 100 / 96], 1.0 + 100 / 192, b)
    # at the expectations, every G_i = 1 and S_i = 100 exactly, so any weights summing to 1 give
    # G = 1, S = 100, B_noise = 100
    assert math.isclose(r["G2"], 1.0, rel_tol=1e-12)
    assert math.isclose(r["trS"], 100.0, rel_tol=1e-12)
    assert math.isclose(r["B_noise"], 100.0, rel_tol=1e-12)


def test_theorem1_matrices_nonsingular_small_clusters():
    """Theorem 1's printed A_G and A_S are nonsingular for EVERY split with n <= 4
    and b_i <= 12 (exact rational determinants, entries retyped from the theorem, not from the
    oracle), so the SINGULAR error is unreachable for such clusters; the oracle's weights exist
    and sum to 1 there."""
    import itertools
    from fractions import Fraction as F

    def det(M):
        M = [row[:] for row in M]
        n, d = len(M), F(1)
        for c in range(n):
            p = next((r for r in range(c, n) if M[r][c] != 0), None)
            if p is None:
                return F(0)
            if p != c:
                M[c], M[p] = M[p], M[c]
                d = -d
            d *= M[c][c]
            for r in range(c + 1, n):
                f = M[r][c] / M[c][c]
                for k in range(c, n):
                    M[r][k] -= f * M[c][k]
        return d

    count = 0
    for n in (2, 3, 4):
        for b in itertools.combinations_with_replacement(range(1, 13), n):
            B = sum(b)
            AG = [[F(B + 2 * b[i], B * B - B * b[i]) if i == j else
                   F(B * B - b[i] ** 2 - b[j] ** 2, B * (B - b[i]) * (B - b[j])) for j in range(n)]
                  for i in range(n)]
            AS = [[F(B * b[i], B - b[i]) if i == j else
                   F(b[i] * b[j] * (B - b[i] - b[j]), (B - b[i]) * (B - b[j])) for j in range(n)]
                  for i in range(n)]
            assert det(AG) != 0 and det(AS) != 0, b
            if count % 97 == 0:
                AGo, ASo = gns.weight_matrices(list(b))
                for A in (AGo, ASo):
                    w = gns.optimal_weights(A)
                    assert np.all(np.isfinite(w)) and abs(float(np.sum(w)) - 1.0) < 1e-12
            count += 1
    assert count == 1807


# ---------------------------------------------------------------- corrected-covariance variant
def _mc_estimates(b, d=128, trials=40_000, G2=1.0, trS=100.0, seed=11):
    """Per-node Eq. 10 estimates over Monte Carlo draws of the paper's model (Eq. 1: g_i = mean of
    b_i iid N(G, Sigma) samples, here drawn directly as N(G, Sigma / b_i)), isotropic Sigma."""
    rng = np.random.default_rng(seed)
    b = np.asarray(b, dtype=float)
    n, B = len(b), float(np.sum(b))
    G = rng.standard_normal(d)
    G *= math.sqrt(G2) / np.linalg.norm(G)
    s2 = trS / d
    Gi = np.empty((trials, n))
    Si = np.empty((trials, n))
    for t0 in range(0, trials, 5000):
        m = min(5000, trials - t0)
        g = G + np.sqrt(s2 / b)[None, :, None] * rng.standard_normal((m, n, d))
        gg = np.einsum("i,tid->td", b / B, g)
        ls = np.einsum("tid,tid->ti", g, g)
        gs = np.einsum("td,td->t", gg, gg)
        for i in range(n):
            Gi[t0:t0 + m, i] = (B * gs - b[i] * ls[:, i]) / (B - b[i])
            Si[t0:t0 + m, i] = b[i] * B / (B - b[i]) * (ls[:, i] - gs)
    tau = 2.0 * d * s2 * s2          # 2 tr(Sigma^2)
    c = 4.0 * s2 * G2                # 4 G^T Sigma G
    return Gi, Si, tau, c


def test_corrected_matrices_match_monte_carlo_covariance():
    """The exact-Gaussian covariance of the Eq. 10 estimators (Isserlis) against the empirical
    covariance of 40k draws of the paper's model at C1's b."""
    b = [32, 64, 96]
    Gi, Si, tau, c = _mc_estimates(b)
    AG, AS = gns.corrected_matrices(b, tau / c)
    for emp, A in ((np.cov(Gi.T) / c, AG), (np.cov(Si.T) / c, AS)):
        scale = np.sqrt(np.outer(np.diag(A), np.diag(A)))
        assert np.max(np.abs(emp - A) / scale) < 0.03, (emp, A)


def test_corrected_weights_minimum_variance_and_unbiased():
    """With the exact covariance the combined estimator is unbiased and has smaller variance than
    both the uniform weights and Theorem 1's printed weights (which lose to uniform at C1's b,
    SURVEY App. A.8)."""
    b = [32, 64, 96]
    Gi, Si, tau, c = _mc_estimates(b, trials=60_000, seed=12)
    AGt, ASt = gns.weight_matrices(b)
    r = gns.gns_estimate_corrected([1.0] * 3, 1.0, b, rho=tau / c)
    variants = {"thm1": (gns.optimal_weights(AGt), gns.optimal_weights(ASt)),
                "uniform": (np.ones(3) / 3, np.ones(3) / 3),
                "corrected": (r["wG"], r["wS"])}
    var = {}
    for k, (wg, ws) in variants.items():
        Ge, Se = Gi @ wg, Si @ ws
        T = len(Ge)
        assert abs(Ge.mean() - 1.0) < 4 * Ge.std() / math.sqrt(T), k
        assert abs(Se.mean() - 100.0) < 4 * Se.std() / math.sqrt(T), k
        var[k] = (Ge.var(), Se.var())
    assert var["corrected"][0] <= var["uniform"][0] * 1.002
    assert var["corrected"][1] < var["uniform"][1] < var["thm1"][1]
    assert var["corrected"][0] < var["thm1"][0]


@pytest.mark.parametrize("b", [[32, 64, 96], [1, 2], [5, 5, 5, 90], [7, 300], [3, 9, 27, 81, 243]])
@pytest.mark.parametrize("rho", [1e-6, 0.5, 50.0, 1e6])
def test_corrected_weights_closed_form(b, rho):
    """A_G (B - b) and A_S (B - b) are constant vectors (shown in DESIGN.md reading Q31), so the
    corrected weights are w_i = (B - b_i) / ((n - 1) B) for G and S, whatever rho; the estimates
    become the pooled forms G = (n B |g|^2 - sum b_i |g_i|^2) / ((n-1) B) and
    S = (sum b_i |g_i|^2 - B |g|^2) / (n - 1)."""
    B, n = sum(b), len(b)
    w = (B - np.asarray(b, float)) / ((n - 1) * B)
    rng = np.random.default_rng(len(b))
    ls = list(1.0 + rng.random(n))
    gs = 1.0 + 0.1 * float(rng.random())
    r = gns.gns_estimate_corrected(ls, gs, b, rho=rho)
    assert np.allclose(r["wG"], w, rtol=0, atol=1e-12) and np.allclose(r["wS"], w, rtol=0, atol=1e-12)
    bl = sum(bi * x for bi, x in zip(b, ls))
    assert math.isclose(r["G2"], (n * B * gs - bl) / ((n - 1) * B), rel_tol=1e-11, abs_tol=1e-12)
    assert math.isclose(r["trS"], (bl - B * gs) / (n - 1), rel_tol=1e-10, abs_tol=1e-10)


def test_corrected_first_order_limit_matches_theorem1_diagonal():
    """At rho -> 0 (the delta-method limit) the corrected A_S diagonal is B b_i / (B - b_i): the
    entry Theorem 1 prints; the off-diagonals differ (reading Q6)."""
    b = [32, 64, 96]
    _, AS0 = gns.corrected_matrices(b, 0.0)
    B = sum(b)
    for i, bi in enumerate(b):
        assert math.isclose(AS0[i, i], B * bi / (B - bi), rel_tol=1e-14)
