"""Pins for oracle/learn.py (the measured-model loop, §4.5) and its library twin."""
import math

import numpy as np
import pytest

import cannikin_synth as synth
import paper_2402_05302_b200 as ck
from oracle import learn
from oracle import optsplit as osp


def test_fit_two_points_solves_the_linear_equations():
    """two local batch sizes determine the line exactly ("solving linear equations")."""
    q, s = 0.0023, 0.041
    slope, icpt = learn.fit_linear([10.0, 30.0], [q * 10 + s, q * 30 + s])
    assert math.isclose(slope, q, rel_tol=1e-12) and math.isclose(icpt, s, rel_tol=1e-12)


def test_fit_noiseless_many_points_and_symmetric_noise():
    xs = [float(x) for x in range(5, 60, 5)]
    ys = [0.5 * x + 3.0 for x in xs]
    sl, ic = learn.fit_linear(xs, ys)
    assert math.isclose(sl, 0.5, rel_tol=1e-13) and math.isclose(ic, 3.0, rel_tol=1e-12)
    # +d, -d noise pairs at the same x leave the least-squares line unchanged
    xs2 = xs + xs
    ys2 = [y + 0.1 for y in ys] + [y - 0.1 for y in ys]
    sl2, ic2 = learn.fit_linear(xs2, ys2)
    assert math.isclose(sl2, 0.5, rel_tol=1e-12) and math.isclose(ic2, 3.0, rel_tol=1e-12)


def test_fit_errors():
    with pytest.raises(ZeroDivisionError):
        learn.fit_linear([1.0], [2.0])
    with pytest.raises(ZeroDivisionError):
        learn.fit_linear([3.0, 3.0], [1.0, 2.0])


def test_ivw_closed_forms():
    """Eq. 12: two nodes -> weight of node 0 is v1/(v0+v1); equal variances -> mean."""
    g = learn.ivw([0.2, 0.4], [1.0, 3.0])
    assert math.isclose(g, 0.2 * 3 / 4 + 0.4 * 1 / 4, rel_tol=1e-15)
    assert math.isclose(learn.ivw([0.1, 0.2, 0.6], [2.0] * 3), 0.3, rel_tol=1e-15)
    assert learn.ivw([0.1, 0.5, 0.3], [0.0, 1.0, 0.0]) == 0.2  # zero variance dominates


def test_min_comm_time_recovers_truth():
    """waiting inflates the faster nodes' T_i; the minimum is the slowest node's, the truth."""
    rng = np.random.default_rng(3)
    nodes, comm = synth.random_cluster(rng, 5)
    obs = synth.simulate_iteration(nodes, comm, [20, 30, 40, 50, 60], rng)
    assert min(o["t_o"] for o in obs) == comm[1] and min(o["t_u"] for o in obs) == comm[2]
    assert max(o["t_o"] for o in obs) > comm[1]


def run_loop(an, nodes, comm, B, epochs, rng, cv=0.0, gamma_sd=None, iters=4):
    plans = []
    it = 0
    for _ in range(epochs):
        p = an.plan(B)
        plans.append(p)
        for _ in range(iters):
            for i, o in enumerate(synth.simulate_iteration(nodes, comm, p["b"], rng, cv, gamma_sd)):
                an.observe(i, it, p["b"][i], o["a"], o["P"], o["gamma"], o["t_o"], o["t_u"])
            it += 1
    return plans


@pytest.mark.parametrize("seed", range(6))
def test_optperf_by_the_third_epoch_noiseless(seed):
    """starting from an even split, OptPerf is reached "as early as the third epoch" -- the
    first two epochs provide the two batch sizes per node the models need."""
    rng = np.random.default_rng(seed)
    n = 4
    nodes, comm = synth.random_cluster(rng, n)
    B = 200
    plans = run_loop(learn.Analyzer(n), nodes, comm, B, 4, rng)
    assert [p["phase"] for p in plans] == [0, 1, 2, 2]
    assert plans[0]["b"] == [50, 50, 50, 50]
    ts = [(nodes[i][0] + nodes[i][2]) * 50 + nodes[i][1] + nodes[i][3] for i in range(n)]
    assert plans[1]["b"] == osp.round_paper(osp.warmup_split([t / 50 for t in ts], B), B)
    b_opt, T_opt = osp.int_split_greedy(nodes, comm, B)
    assert plans[2]["b"] == b_opt and plans[3]["b"] == b_opt
    assert math.isclose(plans[2]["T_pred"], T_opt, rel_tol=1e-9)


def test_noisy_loop_prediction_error_small():
    """§5.3 analog: with 2% timing noise and node-specific gamma noise, the predicted
    OptPerf is within a few percent of the true cluster time of the planned split."""
    rng = np.random.default_rng(11)
    n = 6
    nodes, comm = synth.random_cluster(rng, n)
    plans = run_loop(learn.Analyzer(n), nodes, comm, 300, 6, rng, cv=0.02,
                     gamma_sd=[0.002, 0.05, 0.01, 0.1, 0.003, 0.02], iters=8)
    last = plans[-1]
    T_true = osp.cluster_time(nodes, comm, last["b"])
    assert abs(last["T_pred"] - T_true) / T_true < 0.05
    b_opt, T_opt = osp.int_split_greedy(nodes, comm, 300)
    assert T_true <= T_opt * 1.03


def test_library_analyzer_matches_oracle():
    """The C++ analyzer (cannikin_analyzer_*) against oracle/learn.py on identical telemetry."""
    for seed in range(8):
        rng = np.random.default_rng(100 + seed)
        n = int(rng.integers(2, 8))
        nodes, comm = synth.random_cluster(rng, n)
        B = int(rng.integers(8 * n, 600))
        lib_an, ora_an = ck.Analyzer(n), learn.Analyzer(n)
        gsd = [float(x) for x in rng.uniform(0.0, 0.05, size=n)]
        it = 0
        for epoch in range(5):
            pl, po = lib_an.plan(B), ora_an.plan(B)
            assert pl["phase"] == po["phase"]
            assert pl["b"] == po["b"], (seed, epoch, pl, po)
            if po["phase"] == 2:
                assert math.isclose(pl["T_pred"], po["T_pred"], rel_tol=1e-9)
                ml, cl = lib_an.models()
                mo, co = ora_an.models()
                assert np.allclose(ml, mo, rtol=1e-9, atol=1e-15)
                assert np.allclose(cl, co, rtol=1e-9, atol=1e-15)
            for _ in range(3):
                obs = synth.simulate_iteration(nodes, comm, po["b"], rng, 0.03, gsd)
                for i, o in enumerate(obs):
                    lib_an.observe(i, it, po["b"][i], o["a"], o["P"], o["gamma"], o["t_o"], o["t_u"])
                    ora_an.observe(i, it, po["b"][i], o["a"], o["P"], o["gamma"], o["t_o"], o["t_u"])
                it += 1


def test_library_fit_and_ivw_match_oracle():
    rng = np.random.default_rng(5)
    for _ in range(100):
        k = int(rng.integers(2, 20))
        x = [float(v) for v in rng.integers(1, 500, size=k)]
        if len(set(x)) < 2:
            continue
        y = [float(v) for v in rng.normal(size=k)]
        a = ck.fit_linear(x, y)
        b = learn.fit_linear(x, y)
        assert np.allclose(a, b, rtol=1e-10, atol=1e-12)
        e = [float(v) for v in rng.uniform(0, 1, size=k)]
        v = [float(w) for w in rng.uniform(0.01, 2, size=k)]
        assert math.isclose(ck.ivw(e, v), learn.ivw(e, v), rel_tol=1e-12)
    with pytest.raises(ck.CannikinError):
        ck.fit_linear([1.0, 1.0], [1.0, 2.0])
    with pytest.raises(ck.CannikinError):
        ck.ivw([1.0], [-1.0])


def test_sample_variance_hand_values():
    """Eq. 12's sample variance (reading Q22: ddof = 1): [1, 2, 3, 4] -> 5/3; [2, 2] -> 0;
    [0, 10] -> 50 (the population variance would give 25)."""
    assert abs(learn.sample_variance([1.0, 2.0, 3.0, 4.0]) - 5.0 / 3.0) <= 1e-15
    assert learn.sample_variance([2.0, 2.0]) == 0.0
    assert learn.sample_variance([0.0, 10.0]) == 50.0
