"""Multi-GPU parity of cannikin_weighted_allreduce (every NVLink kernel variant) and of
cannikin_weighted_allreduce_nccl (K4) against the oracle,
bitwise identity across ranks, run-to-run determinism, staging path, multi-bucket stats.
Runs tests/mp_allreduce_worker.py under torchrun on every visible GPU (2..8)."""
import os
import socket
import subprocess
import sys
import tempfile

import numpy as np
import pytest

torch = pytest.importorskip("torch")
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from launch import run_torchrun  # noqa: E402

pytestmark = pytest.mark.gpu

import cannikin_synth as synth  # noqa: E402
from oracle import aggregate as agg  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import mp_allreduce_worker as W  # noqa: E402

TOL = {"f32": 1e-5, "bf16": 1e-2}


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module", params=["static", "dyn", "push", "ll", "ll128", "nccl"])
def results(request):
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    world = min(torch.cuda.device_count(), 8)
    d = tempfile.mkdtemp()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr=127.0.0.1", f"--master-port={_port()}",
           os.path.join(os.path.dirname(__file__), "mp_allreduce_worker.py"), "--out", d]
    env = dict(os.environ, CANNIKIN_SPIN_TIMEOUT_MS="20000",
               CANNIKIN_AR_DYN="1" if request.param == "dyn" else "0",
               CANNIKIN_AR_PUSH="1" if request.param == "push" else "0",
               # "ll": buckets <= 1 MiB / (W-1) through the low-latency kernel (no heap bucket needed)
               CANNIKIN_AR_LL="1" if request.param == "ll" else "0",
               # "ll128": every bucket up to 64 MiB (all but the 355M full-size case) through the
               # flag-in-line two-shot kernel
               CANNIKIN_AR_LL128="1" if request.param == "ll128" else "0",
               CANNIKIN_LL128_MAX_MB="64",
               # "nccl": the cases through cannikin_weighted_allreduce_nccl (K4: NCCL
               # reduce-scatter / all-gather with fused pre/post kernels)
               CANNIKIN_TEST_PATH="nccl" if request.param == "nccl" else "p2p")
    r = run_torchrun(cmd, capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    return world, d


@pytest.mark.parametrize("case", W.CASES, ids=[c[0] for c in W.CASES])
def test_parity_and_identity(results, case):
    world, d = results
    name, N, dtype, seed = case
    ranks = [dict(np.load(os.path.join(d, f"rank{r}_{name}.npz"))) for r in range(world)]
    b = [int(x) for x in ranks[0]["b"]]
    gs = synth.gns_gradients(world, N, b, seed=seed, dtype=dtype)
    r = agg.ratios(b)
    g_ref, ls_ref, gsq_ref = agg.aggregate(gs, r, dtype)
    scale = np.maximum(agg.elementwise_scale([agg.to_f64(g, dtype) for g in gs], r), 1e-30)
    for k in ("out1", "out2", "out3", "out4"):
        got = agg.to_f64(ranks[0][k], dtype)
        err = np.max(np.abs(got - g_ref) / scale) if N else 0.0
        assert err <= TOL[dtype], (k, err)
        for q in range(1, world):  # bitwise identical on every rank
            assert np.array_equal(ranks[q][k], ranks[0][k]), (k, q)
    # the two zero-copy runs are bitwise identical (determinism)
    assert np.array_equal(ranks[0]["out1"], ranks[0]["out2"])
    for sfx in ("", "2", "3", "4", "5"):  # 5: out-of-place cannikin_gns_stats_bucket
        loc, glob = ranks[0]["loc" + sfx], float(ranks[0]["glob" + sfx])
        assert np.allclose(loc, ls_ref, rtol=1e-4, atol=0), (sfx, loc, ls_ref)
        assert abs(glob - gsq_ref) <= 1e-4 * max(gsq_ref, 1e-300), (sfx, glob, gsq_ref)
        for q in range(1, world):
            assert np.array_equal(ranks[q]["loc" + sfx], loc)
            assert float(ranks[q]["glob" + sfx]) == glob
    assert np.array_equal(ranks[0]["loc"], ranks[0]["loc2"])
    assert float(ranks[0]["glob"]) == float(ranks[0]["glob2"])
    assert all(bool(ranks[q]["same5"]) for q in range(world))  # out-of-place: bucket unchanged


def test_ddp_baseline_mean(results):
    world, d = results
    x = np.load(os.path.join(d, "rank0_ddp.npy"))
    assert np.allclose(x, (world + 1) / 2)


def test_probe_then_reduce(results):
    """cannikin_probe_a2a_write (the bench's live NVLink ceiling) runs collectively and a reduction
    right after it is correct: mean of rank+1 over the ranks."""
    world, d = results
    for r in range(world):
        x = np.load(os.path.join(d, f"rank{r}_probe.npy"))
        assert np.allclose(x, (world + 1) / 2, rtol=1e-6)


def test_no_out_of_bounds_writes(results):
    """Guard bands around heap buckets (compute-sanitizer is closed on this pool)."""
    world, d = results
    for N in (1, 7, 4099, (1 << 20) + 3):
        for dtype in ("f32", "bf16"):
            for r in range(world):
                assert bool(np.load(os.path.join(d, f"rank{r}_canary_{dtype}_{N}.npy"))[0]), (N, dtype, r)


def test_check_ratios(results):
    """CANNIKIN_INIT_CHECK_RATIOS: a split whose shares sum to 0.95 is reported as
    DOMAIN by gns_stats on every rank, the reduction still runs (all-ones input -> 0.95), and the
    condition is cleared by the report; correct splits pass."""
    world, d = results
    for r in range(world):
        st = np.load(os.path.join(d, f"rank{r}_check_ratios.npy"))
        assert list(st) == ["OK", "DOMAIN", "OK"], (r, st)
        val = np.load(os.path.join(d, f"rank{r}_check_ratios_val.npy"))
        assert np.allclose(val, [1.0, 0.95, 1.0], rtol=1e-6), (r, val)


def test_result_bits_independent_of_variant():
    """Every K3 variant (static / dynamic pull, static / dynamic push, one-shot, LL) sums
    fmaf(r_j, g_j, acc) in rank order in fp32 and rounds once: identical result bits."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    world = min(torch.cuda.device_count(), 8)
    d = tempfile.mkdtemp()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr=127.0.0.1", f"--master-port={_port()}",
           os.path.join(os.path.dirname(__file__), "mp_allreduce_worker.py"), "--out", d,
           "--variants"]
    r = run_torchrun(cmd, capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, CANNIKIN_SPIN_TIMEOUT_MS="20000"))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    for dtype in ("f32", "bf16"):
        ref = np.load(os.path.join(d, f"rank0_var_static_{dtype}.npy"))
        for name in ("static", "dyn", "push", "ll", "ll128"):
            for k in range(world):
                got = np.load(os.path.join(d, f"rank{k}_var_{name}_{dtype}.npy"))
                assert np.array_equal(got, ref), (name, dtype, k)


@pytest.mark.parametrize("gated", [False, True], ids=["plain", "gated"])
def test_mixed_sequence_of_sizes_dtypes_and_variants(gated):
    """40 calls of seeded random size (1 .. 5M elements), dtype and buffer kind (heap bucket or
    staged tensor) on ONE ctx under the automatic variant choice: every result matches the oracle,
    is bitwise identical on every rank, and every call's statistics match the oracle.  `gated`:
    the same with CANNIKIN_INIT_GATED_ENTRY while a different rank arrives 2 ms late at every call
    (the one-warp gate holds the wait); one extra launch per call is counted."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    world = min(torch.cuda.device_count(), 8)
    d = tempfile.mkdtemp()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr=127.0.0.1", f"--master-port={_port()}",
           os.path.join(os.path.dirname(__file__), "mp_allreduce_worker.py"), "--out", d, "--mixed"]
    if gated:
        cmd.append("--gated")
    r = run_torchrun(cmd, capture_output=True, text=True, timeout=900,
                       env=dict(os.environ, CANNIKIN_SPIN_TIMEOUT_MS="20000"))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    for t in range(W.MIXED_CALLS):
        ranks = [dict(np.load(os.path.join(d, f"rank{k}_mixed_{t}.npz"))) for k in range(world)]
        N, dtype = int(ranks[0]["N"]), str(ranks[0]["dtype"])
        b = [int(x) for x in ranks[0]["b"]]
        gs = synth.gns_gradients(world, N, b, seed=200 + t, dtype=dtype)
        rr = agg.ratios(b)
        g_ref, ls_ref, gsq_ref = agg.aggregate(gs, rr, dtype)
        scale = np.maximum(agg.elementwise_scale([agg.to_f64(g, dtype) for g in gs], rr), 1e-30)
        got = agg.to_f64(ranks[0]["out"], dtype)
        assert np.max(np.abs(got - g_ref) / scale) <= TOL[dtype], (t, N, dtype)
        assert np.allclose(ranks[0]["loc"], ls_ref, rtol=1e-4, atol=0), (t, N)
        assert abs(float(ranks[0]["glob"]) - gsq_ref) <= 1e-4 * max(gsq_ref, 1e-300), (t, N)
        for k in range(1, world):
            assert np.array_equal(ranks[k]["out"], ranks[0]["out"]), (t, k)
            assert np.array_equal(ranks[k]["loc"], ranks[0]["loc"]), (t, k)
        # launches of the call: the reduction (+ 2 staging copies) (+ the gate kernel)
        assert int(ranks[0]["launches"]) in ((2, 4) if gated else (1, 3)), (t, ranks[0]["launches"])
    for k in range(world):  # graph-captured reductions, replayed (late rank when gated)
        ok = np.load(os.path.join(d, f"rank{k}_graph_replays.npy"))
        assert ok.size == 9 and ok.all(), (k, ok)
