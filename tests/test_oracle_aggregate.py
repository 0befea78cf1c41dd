"""Pins for oracle/aggregate.py (Eq. 9 and the Eq. 10 norm inputs) against things other than itself."""
import math

import numpy as np
import pytest

import cannikin_synth as synth
from oracle import aggregate as agg


def test_equal_batches_reduce_to_plain_mean():
    """Eq. 2: with equal b_i the weighted aggregate is the plain average (north-star check 1)."""
    gs = synth.gns_gradients(4, 4099, [16, 16, 16, 16], seed=3)
    gs64 = [agg.to_f64(g, "f32") for g in gs]
    g = agg.weighted_sum(gs64, agg.ratios([16] * 4))
    mean = np.mean(np.stack(gs64), axis=0)
    assert np.max(np.abs(g - mean)) <= 1e-15 * np.max(np.abs(mean)) * 4


def test_one_hot_ratio_selects_rank_exactly():
    gs = synth.gns_gradients(3, 1000, [1, 1, 1], seed=5)
    gs64 = [agg.to_f64(g, "f32") for g in gs]
    g = agg.weighted_sum(gs64, [0.0, 1.0, 0.0])
    assert np.array_equal(g, gs64[1])


def test_per_sample_construction_equals_global_mean():
    """for per-sample means g_i (Eq. 1), Eq. 9 equals the mean of all B per-sample gradients."""
    b = [3, 7, 11, 2]
    G, xs = synth.per_sample_gradients(b, 64, seed=1)
    gi = [x.mean(axis=0) for x in xs]
    g = agg.weighted_sum(gi, agg.ratios(b))
    ref = np.concatenate(xs, axis=0).mean(axis=0)
    assert np.max(np.abs(g - ref)) < 1e-12


def test_wrong_ratio_would_be_caught():
    """Sanity of the pin above: the homogeneous 1/n average differs for unequal b."""
    b = [3, 7, 11, 2]
    _, xs = synth.per_sample_gradients(b, 64, seed=1)
    gi = [x.mean(axis=0) for x in xs]
    ref = np.concatenate(xs, axis=0).mean(axis=0)
    assert np.max(np.abs(agg.weighted_sum(gi, [0.25] * 4) - ref)) > 1e-3


def test_linearity_in_r():
    gs = synth.gns_gradients(3, 513, [1, 2, 3], seed=2)
    gs64 = [agg.to_f64(g, "f32") for g in gs]
    r1, r2 = np.array([0.2, 0.3, 0.5]), np.array([0.6, 0.1, 0.3])
    lhs = agg.weighted_sum(gs64, 0.5 * r1 + 0.5 * r2)
    rhs = 0.5 * agg.weighted_sum(gs64, r1) + 0.5 * agg.weighted_sum(gs64, r2)
    assert np.max(np.abs(lhs - rhs)) < 1e-14


def test_norms_match_fsum_exactly_rounded():
    gs = synth.gns_gradients(3, 1 << 14, [32, 64, 96], seed=0)
    for g in gs:
        x = agg.to_f64(g, "f32")
        assert math.isclose(agg.sq_norm(x), agg.sq_norm_exact(x), rel_tol=1e-13)


def test_zero_noise_norms_equal_G2():
    """trS = 0 => |g_i|^2 = |g|^2 = |G|^2."""
    gs = synth.gns_gradients(3, 1 << 12, [32, 64, 96], G2=2.5, trS=0.0, seed=0)
    _, local_sq, global_sq = agg.aggregate(gs, agg.ratios([32, 64, 96]), "f32")
    # the fp32 cast of G perturbs the norm by <= ~1e-7 relative
    assert np.allclose(local_sq, 2.5, rtol=1e-6)
    assert math.isclose(global_sq, 2.5, rel_tol=1e-6)


@pytest.mark.parametrize("bi", [4, 16])
def test_expected_norm_closed_form(bi):
    """E|g_est|^2 = |G|^2 + tr(Sigma)/b, checked by Monte Carlo within 4 standard errors."""
    d, trials = 128, 4000
    rng = np.random.default_rng(11)
    G = rng.standard_normal(d)
    G *= np.sqrt(1.0 / (G @ G))
    trS = 10.0
    vals = []
    for _ in range(trials):
        xs = G + np.sqrt(trS / d) * rng.standard_normal((bi, d))
        vals.append(agg.sq_norm(xs.mean(axis=0)))
    vals = np.array(vals)
    se = vals.std(ddof=1) / np.sqrt(trials)
    assert abs(vals.mean() - (1.0 + trS / bi)) < 4 * se


def test_bf16_upconversion_exact():
    x = np.array([1.0, -2.5, 3.140625, 1e-3, 65504.0], dtype=np.float32)
    bits = synth.f32_to_bf16_bits(x)
    back = agg.to_f64(bits, "bf16")
    # bf16 has 8 significant bits: values representable in 8 bits round-trip exactly
    assert back[0] == 1.0 and back[1] == -2.5 and back[2] == 3.140625
    assert abs(back[3] - 1e-3) <= 2 ** -8 * 1e-3
    assert abs(back[4] - 65504.0) <= 2 ** -8 * 65504.0


def test_bf16_round_to_nearest_even():
    # 1 + 2^-8 is exactly halfway between bf16 1.0 and 1+2^-7: ties to even -> 1.0
    x = np.array([1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8], dtype=np.float32)
    back = agg.to_f64(synth.f32_to_bf16_bits(x), "bf16")
    assert back[0] == 1.0 and back[1] == 1.0 + 2 ** -6


def test_elementwise_scale_hand_values():
    """Pin of the error-metric denominator (reading Q1): sum_i |r_i g_i[e]| per element, by hand.
    r = (0.25, 0.75), g_0 = (2, 4, 0), g_1 = (-1, 4, -8):
      e=0: |0.25*2| + |0.75*(-1)| = 0.5 + 0.75 = 1.25   (a plain |sum| would give 0.25)
      e=1: 1 + 3 = 4                                    (no cancellation: equals |sum|)
      e=2: 0 + 6 = 6                                    (one rank zero)
    Catches: a dropped r (|g_0|+|g_1| = 3), a max over ranks (0.75), |sum| (0.25), or the sum
    without abs (-0.25)."""
    g0 = np.array([2.0, 4.0, 0.0])
    g1 = np.array([-1.0, 4.0, -8.0])
    s = agg.elementwise_scale([g0, g1], [0.25, 0.75])
    assert s.tolist() == [1.25, 4.0, 6.0]


def test_elementwise_scale_bounds_the_aggregate():
    """Triangle inequality: |sum_i r_i g_i[e]| <= scale[e], with equality where all terms share a
    sign; scale is linear in |r| (doubling r doubles it) and independent of the sign of r_i."""
    gs = synth.gns_gradients(4, 4099, [3, 5, 7, 9], seed=8)
    gs64 = [agg.to_f64(g, "f32") for g in gs]
    r = agg.ratios([3, 5, 7, 9])
    s = agg.elementwise_scale(gs64, r)
    g = agg.weighted_sum(gs64, r)
    assert np.all(np.abs(g) <= s * (1 + 1e-15))
    same = np.all(np.stack(gs64) > 0, axis=0) | np.all(np.stack(gs64) < 0, axis=0)
    assert same.any()
    assert np.allclose(np.abs(g[same]), s[same], rtol=1e-14)
    assert np.allclose(agg.elementwise_scale(gs64, 2 * r), 2 * s, rtol=1e-15)
    assert np.array_equal(agg.elementwise_scale(gs64, -r), s)
