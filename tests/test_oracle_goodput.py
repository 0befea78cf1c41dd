"""Pins for oracle/goodput.py (adaptive total batch, NEXT-2) and its library twin."""
import math

import numpy as np
import pytest

import cannikin_synth as synth
import paper_2402_05302_b200 as ck
from oracle import goodput as ogp
from oracle import learn
from oracle import optsplit as osp

CANDS = [16, 32, 64, 96, 128, 192, 256, 384, 512]


def test_efficiency_closed_forms():
    assert ogp.efficiency(32, 32, 123.0) == 1.0                       # B = B0
    assert math.isclose(ogp.efficiency(512, 32, 1e15), 1.0, rel_tol=1e-12)  # noise dominates
    assert math.isclose(ogp.efficiency(512, 32, 0.0), 32 / 512)       # no noise: B0 / B
    assert math.isclose(ck.efficiency(100, 32, 50.0), ogp.efficiency(100, 32, 50.0), rel_tol=1e-15)


def test_choice_limits():
    """B_noise = 0: goodput = B0 / T(B), T increasing -> the smallest candidate; B_noise -> inf:
    goodput = throughput -> the candidate with the largest B / T(B)."""
    rng = np.random.default_rng(1)
    nodes, comm = synth.random_cluster(rng, 4)
    assert ogp.choose_batch(nodes, comm, CANDS, 32, 0.0) == CANDS[0]
    thr = [B / osp.int_split_greedy(nodes, comm, B)[1] for B in CANDS]
    assert ogp.choose_batch(nodes, comm, CANDS, 32, 1e15) == CANDS[int(np.argmax(thr))]


def test_choice_grows_with_noise_scale():
    """fig:gns: as the GNS grows during training, the chosen total batch grows."""
    rng = np.random.default_rng(2)
    nodes, comm = synth.random_cluster(rng, 4)
    picks = [ogp.choose_batch(nodes, comm, CANDS, 16, bn) for bn in (1, 10, 100, 1000, 1e5)]
    assert picks == sorted(picks) and picks[0] < picks[-1]


def test_ema_separately_not_ratio():
    e = ogp.Ema(0.5)
    e.update(1.0, 100.0)
    e.update(3.0, 100.0)
    assert e.B_noise == 100.0 / 2.0                 # not mean(100, 33.3)
    e.update(-1.0, 5.0)                             # non-positive G skipped (reading Q26)
    assert e.count == 2
    # the worked example above by hand: G = 0.5*1 + 0.5*3 = 2, S = 100 -> 50
    assert e.G2 == 2.0 and e.trS == 100.0


@pytest.mark.parametrize("decay", [0.0, 0.5, 0.9, 0.99])
def test_library_ema_matches_oracle(decay):
    """cannikin_gns_ema_update (library, which also sets B_noise) against the oracle's Ema over a
    seeded sequence of snapshots with non-positive G's mixed in: the same averages, count and
    B_noise = S / G of the averages (reading Q26); NaN before the first accepted one."""
    rng = np.random.default_rng(int(decay * 100))
    le, oe = ck.GnsEma(decay), ogp.Ema(decay)
    assert math.isnan(le.B_noise) and le.count == 0
    le.update(-1.0, 3.0)
    assert math.isnan(le.B_noise) and le.count == 0  # skipped snapshot: still none
    for _ in range(200):
        G = float(rng.normal(1.0, 0.7))
        S = float(rng.uniform(10.0, 500.0))
        le.update(G, S)
        oe.update(G, S)
        assert le.count == oe.count
        if oe.count:
            assert le.B_noise == oe.B_noise


@pytest.mark.parametrize("seed", range(5))
def test_library_choose_batch_matches_oracle(seed):
    rng = np.random.default_rng(10 + seed)
    nodes, comm = synth.random_cluster(rng, int(rng.integers(2, 8)))
    for bn in (0.5, 20.0, 300.0, 4000.0, 1e6):
        r = ck.choose_batch(nodes, comm, CANDS, 16, bn)
        assert r["B"] == ogp.choose_batch(nodes, comm, CANDS, 16, bn)
        for B, T in zip(CANDS, r["T"]):
            assert T == osp.int_split_greedy(nodes, comm, B)[1]


def test_analyzer_choose_batch_cache_equals_brute_force_with_fixed_models():
    """The OptPerf_init cache picks the brute-force optimum when the learned models do
    not change between epochs, and recomputes only when the overlap pattern changes."""
    rng = np.random.default_rng(21)
    n = 4
    nodes, comm = synth.random_cluster(rng, n)
    an = ck.Analyzer(n)
    it = 0
    for b in ([20] * n, [35, 28, 24, 18]):  # two batch sizes per node, noiseless
        for o_i, o in enumerate(synth.simulate_iteration(nodes, comm, b, rng)):
            an.observe(o_i, it, b[o_i], o["a"], o["P"], o["gamma"], o["t_o"], o["t_u"])
        it += 1
    learned, lcomm = an.models()
    fulls = []
    for bn in (1.0, 10.0, 100.0, 1000.0, 1e4, 1e4):
        r = an.choose_batch(CANDS, 16, bn)
        fulls.append(r["full_recompute"])
        assert r["B"] == ogp.choose_batch(learned, lcomm, CANDS, 16, bn)
        assert sum(r["b"]) == r["B"]
    assert fulls[0] is True and fulls[-1] is False


def test_goodput_hand_value():
    """goodput(B) = B / T(B) x efficiency (reading Q27), T = Eq. 7 at the integer split.
    One node with f(b) = 0.01 b (q = 0.01, other terms 0, gamma = 0): B = 100 -> T = 1.0 s,
    throughput 100/s; B0 = 20, B_noise = 80 -> efficiency (80+20)/(80+100) = 5/9 -> 55.5...; also
    T is returned as the second value."""
    g, T = ogp.goodput([(0.01, 0.0, 0.0, 0.0)], (0.0, 0.0, 0.0), 100, 20, 80.0)
    assert abs(T - 1.0) <= 1e-15
    assert abs(g - 100.0 * 5.0 / 9.0) <= 1e-12
