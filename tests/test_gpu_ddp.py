"""End-to-end Eq. 9 through torch DDP with the Cannikin comm hook (NEXT-3): with uneven local
batches b_i and per-rank mean losses, every rank's reduced gradient equals the full-batch mean
gradient over all B samples, bit-identical across ranks; the hook's statistics equal the
local and global squared norms."""
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

from oracle import aggregate as agg  # noqa: E402

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(world):
    d = tempfile.mkdtemp()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr=127.0.0.1", f"--master-port={_port()}",
           os.path.join(os.path.dirname(__file__), "mp_ddp_worker.py"), "--out", d]
    r = run_torchrun(cmd, capture_output=True, text=True, timeout=900,
                       env=dict(os.environ, CANNIKIN_SPIN_TIMEOUT_MS="20000"))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    return [dict(np.load(os.path.join(d, f"rank{k}.npz"))) for k in range(world)]


def _check_oracle(ranks):
    """Every rank's hook result against the oracle's Eq. 9 of the ranks' local gradients (Q1
    metric, fp32 1e-5) and the hook statistics against the oracle's norms (1e-4)."""
    b = [int(x) for x in ranks[0]["b"]]
    gs = [rk["gi"] for rk in ranks]
    r = agg.ratios(b)
    g_ref, ls_ref, gsq_ref = agg.aggregate(gs, r, "f32")
    scale = np.maximum(agg.elementwise_scale([agg.to_f64(g, "f32") for g in gs], r), 1e-30)
    for rk in ranks:
        err = np.max(np.abs(rk["got"].astype(np.float64) - g_ref) / scale)
        assert err <= 1e-5, err
        for key_l, key_g in (("loc", "glob"), ("hook_loc", "hook_glob")):
            assert np.allclose(rk[key_l], ls_ref, rtol=1e-4, atol=0), (key_l, rk[key_l], ls_ref)
            assert abs(float(rk[key_g]) - gsq_ref) <= 1e-4 * gsq_ref


def test_ddp_hook_single_gpu():
    """World 1 (the driver's one-GPU run): the hook's reduction is K2 with r = 1 -- the result is
    the local gradient, the statistics its norm, read both after a host sync and through
    CannikinHookState.gns_stats() -- against the oracle."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    ranks = _run(1)
    assert int(ranks[0]["buckets"]) >= 2
    assert np.array_equal(ranks[0]["got"], ranks[0]["gi"])  # r = 1: g = fmaf(1, g_0, 0) exactly
    _check_oracle(ranks)


def test_ddp_hook_equals_full_batch_gradient():
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    world = min(torch.cuda.device_count(), 8)
    ranks = _run(world)
    _check_oracle(ranks)
    ref = ranks[0]["ref"].astype(np.float64)
    scale = np.max(np.abs(ref))
    for k in range(world):
        assert int(ranks[k]["buckets"]) >= 2          # several DDP buckets went through the hook
        assert int(ranks[k]["buckets"]) == int(ranks[0]["buckets"])
        got = ranks[k]["got"].astype(np.float64)
        assert np.max(np.abs(got - ref)) <= 1e-4 * scale
        assert np.array_equal(ranks[k]["got"], ranks[0]["got"])
        assert np.array_equal(ranks[k]["loc"], ranks[0]["loc"])
        assert abs(float(ranks[0]["loc"][k]) - float(ranks[k]["gi_sq"])) <= 1e-4 * float(ranks[k]["gi_sq"])
    gsq = float((ref ** 2).sum())
    assert abs(float(ranks[0]["glob"]) - gsq) <= 1e-4 * gsq
