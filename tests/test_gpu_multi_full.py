"""Multi-GPU parity at full size in the bench launch configuration (zero-copy heap bucket, default
grid) for configs[3] (110M bf16) and configs[4] (355M fp32, one 1.42 GB bucket): sampled elements
against the oracle one by one, the norm statistics against the oracle over the whole vectors,
identical statistics on every rank."""
import glob
import os
import shutil
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

from oracle import aggregate as agg  # noqa: E402


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


TOL = {"c4": ("bf16", 1e-2), "c5": ("f32", 1e-5)}


@pytest.mark.parametrize("cfg", ["c4", "c5"])
def test_full_size_multi(cfg):
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    world = min(torch.cuda.device_count(), 8)
    d = tempfile.mkdtemp()
    try:
        _run_and_check(cfg, world, d)
    finally:
        shutil.rmtree(d, ignore_errors=True)  # the whole inputs: up to 5.7 GB


def _run_and_check(cfg, world, d):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr=127.0.0.1", f"--master-port={_port()}",
           os.path.join(os.path.dirname(__file__), "mp_allreduce_worker.py"), "--out", d, "--full", cfg]
    r = run_torchrun(cmd, capture_output=True, text=True, timeout=900,
                       env=dict(os.environ, CANNIKIN_SPIN_TIMEOUT_MS="20000"))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    ranks = [dict(np.load(os.path.join(d, f"rank{k}_full.npz"))) for k in range(world)]
    b = [int(x) for x in ranks[0]["b"]]
    rr = agg.ratios(b)
    dt, tol = TOL[cfg]
    ins = [agg.to_f64(x, dt) for x in ranks[0]["ins"]]
    ref = agg.weighted_sum(ins, rr)
    scale = np.maximum(agg.elementwise_scale(ins, rr), 1e-30)
    for k in range(world):
        got = agg.to_f64(ranks[k]["out"], dt)
        assert np.max(np.abs(got - ref) / scale) <= tol
        assert np.array_equal(ranks[k]["loc"], ranks[0]["loc"])
        assert float(ranks[k]["glob"]) == float(ranks[0]["glob"])
    lsum = np.zeros(world)
    gsum = 0.0
    for f in sorted(glob.glob(os.path.join(d, "full_in_*.npy"))):
        parts = [agg.to_f64(x, dt) for x in np.load(f)]
        for j in range(world):
            lsum[j] += agg.sq_norm(parts[j])
        gsum += agg.sq_norm(agg.weighted_sum(parts, rr))
    assert np.allclose(ranks[0]["loc"], lsum, rtol=1e-4)
    assert abs(float(ranks[0]["glob"]) - gsum) <= 1e-4 * gsum
