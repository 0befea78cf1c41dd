"""Pins for oracle/optsplit.py and oracle/pipeline.py against SPEC/paper hand values, the event
pipeline, brute force, KKT equal-time conditions and grid search."""
import math

import numpy as np
import pytest

import cannikin_synth as synth
from oracle import optsplit as osp
from oracle import pipeline


def test_eq3_to_eq6_hand_values(golden):
    ex = golden["node_model"]
    node, b = ex["node"], ex["b"]
    assert math.isclose(osp.compute_time(node, b), ex["compute_time"], rel_tol=1e-12)
    assert math.isclose(osp.sync_start(node, (ex["gamma"], 0, 0), b), ex["sync_start"], rel_tol=1e-12)
    assert math.isclose(osp.node_time(node, ex["compute_bound_comm"], b), ex["compute_bound_time"], rel_tol=1e-12)
    assert osp.is_compute_bound(node, ex["compute_bound_comm"], b)
    assert math.isclose(osp.node_time(node, ex["comm_bound_comm"], b), ex["comm_bound_time"], rel_tol=1e-12)
    assert not osp.is_compute_bound(node, ex["comm_bound_comm"], b)
    ex2 = golden["compute_time_2"]
    assert math.isclose(osp.compute_time(ex2["node"], ex2["b"]), ex2["compute_time"], rel_tol=1e-12)
    ex3 = golden["classify_comm"]
    assert osp.is_compute_bound(ex3["node"], ex3["comm"], ex3["b"]) == ex3["compute_bound"]


def test_classification_tie_is_compute():
    """P:191 '>=': (1-gamma) P == T_o counts as compute-bound."""
    node = (0.0, 0.0, 0.01, 0.0)
    assert osp.is_compute_bound(node, (0.5, 0.25, 0.0), 50)   # (0.5)(0.5) = 0.25


def test_pipeline_spec_traces(golden):
    for ex in golden["pipeline"]:
        T = pipeline.simulate([ex["node"]], ex["comm"], [ex["b"]], ex["n_buckets"])
        assert math.isclose(T, ex["T"], rel_tol=1e-12)


def test_closed_form_equals_pipeline_and_eq7():
    """A.2 / S:490: the bucket pipeline of §3.2.3 equals Eq. 7 = max_i f_i(b_i) for any parameters."""
    rng = np.random.default_rng(7)
    for _ in range(500):
        n = int(rng.integers(1, 9))
        nodes, comm = synth.random_cluster(rng, n)
        b = rng.integers(0, 200, size=n).astype(float)
        nb = int(rng.integers(2, 12))
        T_pipe = pipeline.simulate(nodes, comm, b, nb)
        T_f = osp.cluster_time(nodes, comm, b)
        assert abs(T_pipe - T_f) <= 1e-12 * max(1.0, T_f)
        assert abs(osp.eq7_time(nodes, comm, b) - T_f) <= 1e-12 * max(1.0, T_f)


def test_check1_all_compute(golden):
    ex = golden["solve_equal_compute"]
    b, T, labels = osp.real_split(ex["nodes"], ex["comm"], ex["B"])
    assert np.allclose(b, ex["b"], rtol=0, atol=1e-9)
    assert math.isclose(T, ex["t"], rel_tol=1e-12)
    assert labels == [1, 1]


def test_check2_all_comm(golden):
    ex = golden["solve_equal_syncstart"]
    b, T, labels = osp.real_split(ex["nodes"], ex["comm"], ex["B"])
    assert np.allclose(b, ex["b"], rtol=0, atol=1e-9)
    gamma, t_o, t_u = ex["comm"]
    assert math.isclose(T - t_o - t_u, ex["sync_start"], rel_tol=1e-12)
    assert labels == [0, 0]
    for i in range(2):
        assert math.isclose(osp.sync_start(ex["nodes"][i], ex["comm"], b[i]), ex["sync_start"], rel_tol=1e-12)


def test_rounding_regression(golden):
    ex = golden["rounding_regression"]
    b, T, _ = osp.real_split(ex["nodes"], ex["comm"], ex["B"])
    assert np.allclose(b, ex["b_real"], atol=1e-12)
    assert math.isclose(T, ex["T_real"], rel_tol=1e-12)
    bp = osp.round_paper(b, ex["B"])
    assert bp == ex["b_paper"]
    assert math.isclose(osp.cluster_time(ex["nodes"], ex["comm"], bp), ex["T_paper"], rel_tol=1e-12)
    bi, Ti = osp.int_split_greedy(ex["nodes"], ex["comm"], ex["B"])
    assert bi == ex["b_int"] and math.isclose(Ti, ex["T_int"], rel_tol=1e-12)


def test_round_paper_spec(golden):
    for ex in golden["round_allocation"]:
        assert osp.round_paper(ex["b_real"], ex["B"]) == ex["b"]


def test_warmup_spec(golden):
    for ex in golden["warmup"]:
        assert np.allclose(osp.warmup_split(ex["t_sample"], ex["B"]), ex["b"], rtol=1e-12)


def test_greedy_equals_brute_force():
    """North-star check 3: the integer split agrees with brute-force enumeration on 2-3 node clusters."""
    rng = np.random.default_rng(2024)
    for trial in range(150):
        n = int(rng.integers(2, 4))
        nodes, comm = synth.random_cluster(rng, n)
        B = int(rng.integers(n, 40 if n == 3 else 60))
        lo = cap = None
        if trial % 5 == 0:
            cap = [int(x) for x in rng.integers(max(1, B // n), B, size=n)]
            if sum(cap) < B:
                cap = None
        bg, Tg = osp.int_split_greedy(nodes, comm, B, lo, cap)
        bb, Tb = osp.int_split_brute(nodes, comm, B, lo, cap)
        assert bg == bb, (nodes, comm, B, bg, bb)
        assert Tg == Tb


def test_brute_force_minimises_eq7():
    """The brute force's primary criterion is Eq. 7 itself: no split has a smaller max finish time."""
    rng = np.random.default_rng(99)
    for _ in range(40):
        nodes, comm = synth.random_cluster(rng, 2)
        B = int(rng.integers(2, 50))
        bb, Tb = osp.int_split_brute(nodes, comm, B)
        best = min(osp.cluster_time(nodes, comm, [j, B - j]) for j in range(1, B))
        assert Tb == best


def test_real_split_equal_finish_times_and_bounds():
    """KKT (App. A): unclamped nodes finish together; the integer optimum lies
    within one sample's slope of the relaxation."""
    rng = np.random.default_rng(5)
    for _ in range(300):
        n = int(rng.integers(2, 9))
        nodes, comm = synth.random_cluster(rng, n)
        B = int(rng.integers(4 * n, 1600))
        b, T, labels = osp.real_split(nodes, comm, B)
        assert abs(sum(b) - B) < 1e-7 * B
        times = [osp.node_time(nodes[i], comm, b[i]) for i in range(n) if b[i] > 1.0]
        if len(times) >= 2:
            assert max(times) - min(times) <= 1e-11 * T
        bi, Ti = osp.int_split_greedy(nodes, comm, B)
        slope = max(q + k for q, s, k, m in nodes)
        assert T <= Ti * (1 + 1e-12) and Ti < T + slope + 1e-12
        # mixed patterns: compute-bound nodes share t_compute, comm-bound share syncStart,
        # t_compute = syncStart + T_o
        gamma, t_o, t_u = comm
        tc = [osp.compute_time(nodes[i], b[i]) for i in range(n) if labels[i] and b[i] > 1.0]
        ss = [osp.sync_start(nodes[i], comm, b[i]) for i in range(n) if not labels[i] and b[i] > 1.0]
        if tc and ss:
            assert abs(tc[0] - (ss[0] + t_o)) <= 1e-10 * T


def test_real_split_beats_grid():
    """Optimality of the relaxation on 2 nodes against a fine grid over b_0."""
    rng = np.random.default_rng(11)
    for _ in range(30):
        nodes, comm = synth.random_cluster(rng, 2)
        B = 100
        b, T, _ = osp.real_split(nodes, comm, B)
        grid = np.linspace(1.0, B - 1.0, 20001)
        Tg = min(osp.cluster_time(nodes, comm, [x, B - x]) for x in grid)
        assert T <= Tg + 1e-12
        assert T >= Tg - 0.01 * max(q + k for q, s, k, m in nodes)


def test_homogeneous_even_split_extra_to_low_ranks():
    nodes = [(0.001, 0.01, 0.002, 0.02)] * 4
    comm = (0.3, 0.05, 0.01)
    b, T = osp.int_split_greedy(nodes, comm, 103)
    assert b == [26, 26, 26, 25]
    br, Tr, _ = osp.real_split(nodes, comm, 100)
    assert np.allclose(br, 25.0, atol=1e-9)


def test_single_node():
    b, T = osp.int_split_greedy([(0.001, 0.01, 0.002, 0.02)], (0.3, 0.05, 0.01), 77)
    assert b == [77]
    br, Tr, _ = osp.real_split([(0.001, 0.01, 0.002, 0.02)], (0.3, 0.05, 0.01), 77)
    assert br == [77.0]


def test_errors():
    nodes = [(0.001, 0.01, 0.002, 0.02)] * 2
    with pytest.raises(ValueError):
        osp.int_split_greedy(nodes, (0.3, 0.05, 0.01), 1)          # sum(lo) = 2 > B
    with pytest.raises(ValueError):
        osp.int_split_greedy(nodes, (1.0, 0.05, 0.01), 10)          # gamma out of [0,1)
    with pytest.raises(ZeroDivisionError):
        osp.int_split_greedy([(0.0, 0.01, 0.0, 0.02)] * 2, (0.3, 0.05, 0.01), 10)
    with pytest.raises(ValueError):
        osp.int_split_greedy(nodes, (0.3, 0.05, 0.01), 10, cap=[3, 3])


# ------------------------------------------------------------- Algorithm 1, literally
def test_algorithm1_checks_hand_values(golden):
    """Alg. 1's Check 1 / Check 2 on SPEC's worked examples."""
    ex = golden["solve_equal_compute"]
    r = osp.algorithm1(ex["nodes"], ex["comm"], ex["B"])
    assert r["case"] == "compute"
    assert np.allclose(r["b"], ex["b"], rtol=1e-12)
    assert math.isclose(r["T"], ex["t"] + ex["comm"][2], rel_tol=1e-12)
    ex = golden["solve_equal_syncstart"]
    r = osp.algorithm1(ex["nodes"], ex["comm"], ex["B"])
    assert r["case"] == "comm"
    assert np.allclose(r["b"], ex["b"], rtol=1e-12)
    assert math.isclose(r["T"], ex["sync_start"] + ex["comm"][1] + ex["comm"][2], rel_tol=1e-12)


def test_algorithm1_counterexample_fixing_rule():
    """node 2 is comm-bound in Check 1 AND Check 2, so Alg. 1 fixes it as
    comm-bound, but at the optimum it is compute-bound -- no boundary is consistent.
    The exact solver finds b = [36.24, 43.53, 11.23], T = 0.532255 with node 2 compute-bound."""
    comm = (0.1351, 0.2802, 0.0504)
    nodes = [(0.0031, 0.0833, 0.0012, 0.001), (0.0015, 0.001, 0.0094, 0.0064),
             (0.0041, 0.0841, 0.0311, 0.0024)]
    assert osp.algorithm1(nodes, comm, 91) is None
    b, T, labels = osp.real_split(nodes, comm, 91, lo=[0, 0, 0])
    assert np.allclose(b, [36.24, 43.53, 11.23], atol=0.01)
    assert abs(T - 0.532255) < 1e-6 and labels[2] == 1


def test_algorithm1_agrees_with_exact_split_whenever_it_answers():
    """On random mixed clusters the literal Alg. 1, when it answers, equals the exact relaxation
    (same b and OptPerf); when it fails, the cause is always the P:310 fixing rule: some node with
    the same state in Check 1 and Check 2 has the other state at the optimum."""
    import random
    rng = random.Random(5)
    answered = failed = 0
    for _ in range(600):
        n = rng.randint(2, 6)
        comm = (rng.uniform(0, 0.9), rng.uniform(0, 0.5), rng.uniform(0, 0.1))
        nodes = [(rng.uniform(1e-4, 5e-3), rng.uniform(0, 0.1), rng.uniform(1e-4, 4e-2),
                  rng.uniform(0, 0.01)) for _ in range(n)]
        B = rng.randint(10 * n, 200)
        b, T, labels = osp.real_split(nodes, comm, B, lo=[0] * n)
        if min(b) <= 1e-9:
            continue  # Alg. 1 works on the unbounded relaxation; skip clamped optima
        r = osp.algorithm1(nodes, comm, B)
        if r is None:
            failed += 1
            lab = []
            for line in ([(q + k, s + m) for q, s, k, m in nodes],
                         [(q + comm[0] * k, s + comm[0] * m) for q, s, k, m in nodes]):
                _, bb = osp._solve_equal(line, B)
                lab.append([osp.is_compute_bound(nodes[i], comm, bb[i]) for i in range(n)])
            assert any(lab[0][i] == lab[1][i] and int(lab[0][i]) != labels[i] for i in range(n))
            continue
        answered += 1
        assert math.isclose(r["T"], T, rel_tol=1e-9)
        assert np.allclose(r["b"], b, rtol=1e-7, atol=1e-7)
    assert answered > 10 * max(failed, 1)


def test_node_inverse_hand_values_and_both_branches():
    """node_inverse = the largest b with f(b) <= T, f = max(compute line, comm line).  Hand example:
    q, s, k, m = 1, 2, 3, 4; gamma = 0.5, T_o = 10, T_u = 1:
      compute line (q+k) b + (s+m+T_u)               = 4 b + 7
      comm line    (q+gamma k) b + (s+gamma m+T_o+T_u) = 2.5 b + 15
    The lines cross at b = 8/1.5 = 16/3 (f = 85/3): below it the comm line binds, above the compute.
    T = 40: compute 33/4 = 8.25, comm 10  -> 8.25 (compute-bound side);
    T = 20: compute 13/4 = 3.25, comm 2   -> 2    (comm-bound side)."""
    node, comm = (1.0, 2.0, 3.0, 4.0), (0.5, 10.0, 1.0)
    assert osp.node_inverse(node, comm, 40.0) == 8.25
    assert osp.node_inverse(node, comm, 20.0) == 2.0
    for T in (20.0, 85.0 / 3.0, 40.0, 123.0):  # f(f^-1(T)) = T on both branches and at the kink
        assert abs(osp.node_time(node, comm, osp.node_inverse(node, comm, T)) - T) <= 1e-12 * T


def test_breakpoint_time_hand_value():
    """T* = f(b_bp) with b_bp = (T_o/(1-gamma) - m)/k where (1-gamma) P = T_o.  Same node:
    b_bp = (10/0.5 - 4)/3 = 16/3, the crossing of the two lines above, f = 4*16/3 + 7 = 85/3; a
    node with k = 0 is compute-bound forever iff (1-gamma) m >= T_o."""
    node, comm = (1.0, 2.0, 3.0, 4.0), (0.5, 10.0, 1.0)
    assert abs(osp.breakpoint_time(node, comm) - 85.0 / 3.0) <= 1e-13
    assert osp.is_compute_bound(node, comm, 16.0 / 3.0 + 1e-9)
    assert not osp.is_compute_bound(node, comm, 16.0 / 3.0 - 1e-9)
    assert osp.breakpoint_time((1.0, 0.0, 0.0, 30.0), comm) == -math.inf   # (1-g) m = 15 >= 10
    assert osp.breakpoint_time((1.0, 0.0, 0.0, 10.0), comm) == math.inf    # 5 < 10
