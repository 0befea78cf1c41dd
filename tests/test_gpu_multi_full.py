"""Multi-GPU parity at full size in the bench launch configuration (zero-copy heap bucket, default
grid) for configs[3] (110M bf16, one bucket, and the bench's 25 MB buckets) and configs[4]
(355M fp32, one 1.42 GB bucket): EVERY element
against the oracle (chunked, in the worker's rank 0; the other ranks' results bitwise equal to
rank 0's), the norm statistics against the oracle over the whole vectors, identical statistics on
every rank."""
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


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


TOL = {"c4": ("bf16", 1e-2), "c5": ("f32", 1e-5), "c4b25": ("bf16", 1e-2)}


@pytest.mark.parametrize("cfg", ["c4", "c5", "c4b25"])
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
    dt, tol = TOL[cfg]
    # rank 0 compared every element of every rank's result with the oracle (tests/parity.py)
    assert float(ranks[0]["max_err"]) <= tol
    for k in range(world):
        assert np.array_equal(ranks[k]["loc"], ranks[0]["loc"])
        assert float(ranks[k]["glob"]) == float(ranks[0]["glob"])
    assert np.allclose(ranks[0]["loc"], ranks[0]["oracle_loc"], rtol=1e-4)
    gsum = float(ranks[0]["oracle_glob"])
    assert abs(float(ranks[0]["glob"]) - gsum) <= 1e-4 * gsum
