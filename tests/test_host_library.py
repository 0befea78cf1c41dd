"""CPU tests of libcannikin.so: it loads, exports every symbol include/cannikin.h declares, and its
host solvers agree with the oracle (opt_split bit-exact, GNS within 1e-12)."""
import math
import os
import re
import subprocess

import numpy as np
import pytest

import cannikin_synth as synth
import paper_2402_05302_b200 as ck
from oracle import goodput as ogp
from oracle import gns as ogns
from oracle import optsplit as osp

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include",
                      "cannikin.h")


def declared_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(cannikin_[a-z_0-9]+)\s*\(", txt)))


def test_library_loads_and_exports_every_declared_symbol():
    L = ck.lib()
    names = declared_symbols()
    assert len(names) >= 17
    for name in names:
        assert hasattr(L, name), name
        assert name in ck.SIGNATURES, name
    out = subprocess.run(["nm", "-D", "--defined-only", ck.lib_path()], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r" T (cannikin_\w+)", out))
    assert set(names) <= exported
    assert ck.lib().cannikin_version() == 10000


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", ck.lib_path()], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


# ----------------------------------------------------------------------------- node time
def test_node_time_bit_exact_vs_oracle():
    rng = np.random.default_rng(3)
    for _ in range(2000):
        nodes, comm = synth.random_cluster(rng, 1)
        b = float(rng.integers(0, 5000))
        assert ck.node_time(nodes[0], comm, b) == osp.node_time(nodes[0], comm, b)


# ----------------------------------------------------------------------------- opt_split
def test_opt_split_golden(golden):
    ex = golden["solve_equal_compute"]
    r = ck.opt_split(ex["nodes"], ex["comm"], ex["B"])
    assert np.allclose(r["b_real"], ex["b"], atol=1e-9)
    assert math.isclose(r["T_real"], ex["t"], rel_tol=1e-12)
    assert r["labels"] == [1, 1]
    ex = golden["solve_equal_syncstart"]
    r = ck.opt_split(ex["nodes"], ex["comm"], ex["B"])
    assert np.allclose(r["b_real"], ex["b"], atol=1e-9)
    assert math.isclose(r["T_real"] - ex["comm"][1] - ex["comm"][2], ex["sync_start"], rel_tol=1e-12)
    assert r["labels"] == [0, 0]
    ex = golden["rounding_regression"]
    r = ck.opt_split(ex["nodes"], ex["comm"], ex["B"])
    assert r["b"] == ex["b_int"] and math.isclose(r["T_int"], ex["T_int"], rel_tol=1e-12)
    assert np.allclose(r["b_real"], ex["b_real"], atol=1e-12)
    rp = ck.opt_split(ex["nodes"], ex["comm"], ex["B"], round_paper=True)
    assert rp["b"] == ex["b_paper"] and math.isclose(rp["T_int"], ex["T_paper"], rel_tol=1e-12)


def test_opt_split_bit_exact_vs_brute_force():
    """North-star check 3 through the library: integer split == brute force, bit for bit."""
    rng = np.random.default_rng(77)
    for trial in range(150):
        n = int(rng.integers(1, 4))
        nodes, comm = synth.random_cluster(rng, n)
        B = int(rng.integers(n, 40 if n == 3 else 60))
        cap = None
        if trial % 4 == 0 and n > 1:
            cap = [int(x) for x in rng.integers(max(1, B // n), B + 1, size=n)]
            if sum(cap) < B:
                cap = None
        r = ck.opt_split(nodes, comm, B, cap=cap)
        bb, Tb = osp.int_split_brute(nodes, comm, B, cap=cap)
        assert r["b"] == bb, (nodes, comm, B, cap)
        assert r["T_int"] == Tb


@pytest.mark.parametrize("n", [2, 3, 5, 8])
def test_opt_split_vs_oracle_greedy_and_bisection(n):
    rng = np.random.default_rng(1000 + n)
    for trial in range(60):
        nodes, comm = synth.random_cluster(rng, n)
        B = int(rng.choice([n, 64, 100, 400, 1600, 5000]))
        B = max(B, n)
        lo = None
        if trial % 3 == 0:
            lo = [int(x) for x in rng.integers(1, 4, size=n)]
            if sum(lo) > B:
                lo = None
        r = ck.opt_split(nodes, comm, B, lo=lo)
        bg, Tg = osp.int_split_greedy(nodes, comm, B, lo=lo)
        assert r["b"] == bg
        assert r["T_int"] == Tg
        br, Tr, lab = osp.real_split(nodes, comm, B, lo=lo)
        assert np.allclose(r["b_real"], br, rtol=0, atol=1e-9 * B)
        assert math.isclose(r["T_real"], Tr, rel_tol=1e-12)
        gamma, t_o, _ = comm
        for i in range(n):
            margin = (1 - gamma) * (nodes[i][2] * br[i] + nodes[i][3]) - t_o
            if abs(margin) > 1e-9:
                assert r["labels"][i] == lab[i]


def test_opt_split_paper_rounding_vs_oracle():
    rng = np.random.default_rng(4)
    checked = 0
    for _ in range(200):
        n = int(rng.integers(2, 8))
        nodes, comm = synth.random_cluster(rng, n)
        B = int(rng.integers(4 * n, 1000))
        br, _, _ = osp.real_split(nodes, comm, B)
        fr = [x - math.floor(x) for x in br]
        if min(abs(a - b) for i, a in enumerate(fr) for b in fr[i + 1:]) < 1e-6:
            continue  # remainder ties are decided by rounding noise; skip them
        if min(min(f, 1 - f) for f in fr) < 1e-6:
            continue
        r = ck.opt_split(nodes, comm, B, round_paper=True)
        assert r["b"] == osp.round_paper(br, B)
        checked += 1
    assert checked > 100


def test_opt_split_large_B_fast_and_exact():
    rng = np.random.default_rng(8)
    nodes, comm = synth.random_cluster(rng, 8)
    B = 200_000
    r = ck.opt_split(nodes, comm, B)
    bg, Tg = osp.int_split_greedy(nodes, comm, B)
    assert r["b"] == bg and r["T_int"] == Tg


def test_opt_split_errors():
    nodes = [(0.001, 0.01, 0.002, 0.02)] * 2
    comm = (0.3, 0.05, 0.01)
    with pytest.raises(ck.CannikinError) as e:
        ck.opt_split(nodes, comm, 1)
    assert e.value.name == "INFEASIBLE"
    with pytest.raises(ck.CannikinError) as e:
        ck.opt_split(nodes, (1.0, 0.05, 0.01), 10)
    assert e.value.name == "DOMAIN"
    with pytest.raises(ck.CannikinError) as e:
        ck.opt_split([(0.0, 0.01, 0.0, 0.02)] * 2, comm, 10)
    assert e.value.name == "SINGULAR"
    with pytest.raises(ck.CannikinError) as e:
        ck.opt_split(nodes, comm, 10, cap=[3, 3])
    assert e.value.name == "INFEASIBLE"
    with pytest.raises(ck.CannikinError) as e:
        ck.opt_split([(-0.001, 0.01, 0.002, 0.02)] * 2, comm, 10)
    assert e.value.name == "DOMAIN"
    with pytest.raises(ck.CannikinError) as e:
        ck.opt_split(nodes, comm, 0)
    assert e.value.name == "INVALID"


def test_opt_split_single_node_and_homogeneous():
    r = ck.opt_split([(0.001, 0.01, 0.002, 0.02)], (0.3, 0.05, 0.01), 77)
    assert r["b"] == [77] and r["b_real"] == [77.0]
    r = ck.opt_split([(0.001, 0.01, 0.002, 0.02)] * 4, (0.3, 0.05, 0.01), 103)
    assert r["b"] == [26, 26, 26, 25]


def test_warmup_split_golden(golden):
    for ex in golden["warmup"]:
        b, br = ck.warmup_split(ex["t_sample"], ex["B"])
        assert np.allclose(br, ex["b"], rtol=1e-12)
        assert b == [int(round(x)) for x in ex["b"]]
        assert np.allclose(br, osp.warmup_split(ex["t_sample"], ex["B"]), rtol=1e-14)


# ----------------------------------------------------------------------------- GNS
def test_gns_estimate_golden(golden):
    ex = golden["local_estimates"]
    r = ck.gns_estimate([ex["local_sq"], 1.0], ex["global_sq"], [ex["b_i"], ex["B"] - ex["b_i"]])
    assert math.isclose(r["Gi"][0], ex["G_i"], rel_tol=1e-15)
    assert math.isclose(r["Si"][0], ex["S_i"], rel_tol=1e-15)


def test_gns_estimate_vs_oracle():
    rng = np.random.default_rng(12)
    for _ in range(300):
        n = int(rng.integers(2, 17))
        b = [int(x) for x in rng.integers(1, 300, size=n)]
        gsq = float(rng.uniform(0.5, 3.0))
        lsq = [gsq + float(rng.uniform(-0.2, 5.0)) for _ in range(n)]
        r = ck.gns_estimate(lsq, gsq, b)
        o = ogns.gns_estimate(lsq, gsq, b)
        assert np.allclose(r["wG"], o["wG"], rtol=1e-9, atol=1e-11)
        assert np.allclose(r["wS"], o["wS"], rtol=1e-9, atol=1e-11)
        assert np.allclose(r["Gi"], o["Gi"], rtol=1e-13, atol=1e-13)
        assert np.allclose(r["Si"], o["Si"], rtol=1e-13, atol=1e-11)
        scaleG = sum(abs(w * g) for w, g in zip(o["wG"], o["Gi"])) + 1e-300
        scaleS = sum(abs(w * s) for w, s in zip(o["wS"], o["Si"])) + 1e-300
        assert abs(r["G2"] - o["G2"]) <= 1e-9 * scaleG
        assert abs(r["trS"] - o["trS"]) <= 1e-9 * scaleS
        assert abs(sum(r["wG"]) - 1) < 1e-12 and abs(sum(r["wS"]) - 1) < 1e-12


def test_gns_estimate_corrected_vs_oracle():
    """The library's closed form against the oracle's general construction (matrix solve)."""
    rng = np.random.default_rng(13)
    for _ in range(300):
        n = int(rng.integers(2, 17))
        b = [int(x) for x in rng.integers(1, 300, size=n)]
        gsq = float(rng.uniform(0.5, 3.0))
        lsq = [gsq + float(rng.uniform(-0.2, 5.0)) for _ in range(n)]
        r = ck.gns_estimate(lsq, gsq, b, corrected=True)
        o = ogns.gns_estimate_corrected(lsq, gsq, b)
        assert np.allclose(r["wG"], o["wG"], rtol=1e-9, atol=1e-11)
        assert np.allclose(r["wS"], o["wS"], rtol=1e-9, atol=1e-11)
        scaleG = sum(abs(w * g) for w, g in zip(o["wG"], o["Gi"])) + 1e-300
        scaleS = sum(abs(w * s) for w, s in zip(o["wS"], o["Si"])) + 1e-300
        assert abs(r["G2"] - o["G2"]) <= 1e-9 * scaleG
        assert abs(r["trS"] - o["trS"]) <= 1e-9 * scaleS
    with pytest.raises(ck.CannikinError) as e:
        ck.gns_estimate([1.0, 1.0], 1.0, [5, 0], corrected=True)
    assert e.value.name == "DOMAIN"


def test_gns_estimate_flags_and_errors():
    r = ck.gns_estimate([5.0, 5.0], 0.0, [10, 10])   # G_i = -5 < 0
    assert r["flags"] & ck.GNS_G_NONPOSITIVE
    for bad_b in ([10], [0, 5], [5, -1]):
        with pytest.raises(ck.CannikinError) as e:
            ck.gns_estimate([1.0] * len(bad_b), 1.0, bad_b)
        assert e.value.name in ("INVALID", "DOMAIN")
    with pytest.raises(ck.CannikinError) as e:
        ck.gns_estimate([float("nan"), 1.0], 1.0, [3, 4])
    assert e.value.name == "DOMAIN"


def test_analyzer_api_errors():
    with pytest.raises(ck.CannikinError):
        ck.Analyzer(0)
    an = ck.Analyzer(2)
    with pytest.raises(ck.CannikinError) as e:
        an.observe(5, 0, 10, 0.1, 0.1, 0.1, 0.0, 0.0)          # node out of range
    assert e.value.name == "INVALID"
    with pytest.raises(ck.CannikinError) as e:
        an.observe(0, 0, 10, -0.1, 0.1, 0.1, 0.0, 0.0)         # negative time
    assert e.value.name == "DOMAIN"
    with pytest.raises(ck.CannikinError) as e:
        an.models()                                            # no data yet
    assert e.value.name == "SINGULAR"
    with pytest.raises(ck.CannikinError) as e:
        an.plan(1)                                             # B < n
    assert e.value.name == "INVALID"
    assert an.plan(9, cap=[3, 9])["b"] == [3, 6]               # caps respected in the even split
    with pytest.raises(ck.CannikinError) as e:
        an.plan(9, cap=[3, 3])
    assert e.value.name == "INFEASIBLE"


def test_emulate_compute_domain():
    with pytest.raises(ck.CannikinError) as e:
        ck.emulate_compute(-1.0)
    assert e.value.name == "DOMAIN"


def test_control_step_matches_parts():
    """cannikin_control_step == gns_estimate + EMA + opt_split called separately."""
    import ctypes
    rng = np.random.default_rng(9)
    for _ in range(20):
        n = int(rng.integers(2, 8))
        b = [int(x) for x in rng.integers(1, 100, size=n)]
        gsq = float(rng.uniform(0.5, 2.0))
        lsq = [gsq + float(rng.uniform(0.0, 3.0)) for _ in range(n)]
        nodes, comm = synth.random_cluster(rng, n)
        Bn = int(rng.integers(n, 500))
        stats = (ctypes.c_double * (n + 1))(*(lsq + [gsq]))
        c = ck.ControlStep(b, nodes, comm, Bn)
        c(ctypes.addressof(stats))
        r = c.result
        e = ck.gns_estimate(lsq, gsq, b)
        assert r["G2"] == e["G2"] and r["trS"] == e["trS"] and r["wS"] == e["wS"]
        assert r["b_next"] == ck.opt_split(nodes, comm, Bn)["b"]
        oe = ogp.Ema(0.9)  # the oracle's EMA (reading Q26) of the same snapshot
        oe.update(e["G2"], e["trS"])
        if e["G2"] > 0:
            assert r["ema_B_noise"] == oe.B_noise
        else:
            assert math.isnan(r["ema_B_noise"]) and oe.count == 0
