"""Parity of the NVSwitch-multicast weighted all-reduce (K6, NEXT-4) against the oracle on 2+
GPUs; identical bits on every rank; statistics."""
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
import mp_nvls_worker as W  # noqa: E402

# fp32: the switch sums fp32 terms; the scaled terms r_j g_j are rounded to fp32 first
TOL = {"f32": 1e-5}


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def results():
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    world = min(torch.cuda.device_count(), 8)
    d = tempfile.mkdtemp()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr=127.0.0.1", f"--master-port={_port()}",
           os.path.join(os.path.dirname(__file__), "mp_nvls_worker.py"), "--out", d]
    r = run_torchrun(cmd, capture_output=True, text=True, timeout=900,
                       env=dict(os.environ, CANNIKIN_SPIN_TIMEOUT_MS="20000"))
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    return world, d


@pytest.mark.parametrize("case", W.CASES, ids=[c[0] for c in W.CASES])
def test_nvls_parity(results, case):
    world, d = results
    name, N, dtype, seed = case
    ranks = [dict(np.load(os.path.join(d, f"rank{r}_{name}.npz"))) for r in range(world)]
    b = [int(x) for x in ranks[0]["b"]]
    gs = synth.gns_gradients(world, N, b, seed=seed, dtype=dtype)
    r = agg.ratios(b)
    g_ref, ls_ref, gsq_ref = agg.aggregate(gs, r, dtype)
    scale = np.maximum(agg.elementwise_scale([agg.to_f64(g, dtype) for g in gs], r), 1e-30)
    for k in ("out1", "out2"):
        got = agg.to_f64(ranks[0][k], dtype)
        assert np.max(np.abs(got - g_ref) / scale) <= TOL[dtype], k
        for q in range(1, world):
            assert np.array_equal(ranks[q][k], ranks[0][k])
    for sfx in ("", "2"):
        loc, glob = ranks[0]["loc" + sfx], float(ranks[0]["glob" + sfx])
        assert np.allclose(loc, ls_ref, rtol=1e-4, atol=0)
        assert abs(glob - gsq_ref) <= 1e-4 * gsq_ref
        for q in range(1, world):
            assert np.array_equal(ranks[q]["loc" + sfx], loc)
            assert float(ranks[q]["glob" + sfx]) == glob


def test_nvls_refuses_ragged_and_bf16(results):
    world, d = results
    for r in range(world):
        assert str(np.load(os.path.join(d, f"rank{r}_ragged.npy"))[0]) == "UNSUPPORTED"
        assert str(np.load(os.path.join(d, f"rank{r}_bf16.npy"))[0]) == "UNSUPPORTED"
