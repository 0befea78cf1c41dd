"""The multi-GPU reduction kernels on ONE GPU: cannikin_init_group_local makes W ranks in this
process (same device, each with its own region, the others' regions as peers), and
cannikin_weighted_allreduce_group runs all W ranks' kernel as ONE launch of W x G CTAs (CTA c
plays rank c / G), so the ranks are co-resident by construction -- exactly the per-rank kernels
W GPUs run, also under a profiler that serialises launches.  Every K3 variant (static / dynamic
pull, push, LL, LL128, and the automatic choice) against the oracle (Eq. 9, Eq. 10 inputs),
bitwise identical results and statistics on every rank, result bits identical across variants,
staged (non-heap) buffers, and the ratio check -- for W = 2, 3, 4 and 8 (the 8-rank protocol,
otherwise only reachable on an 8-GPU box).  One test also issues the per-rank
cannikin_weighted_allreduce calls on W concurrent streams (the multi-process call pattern).  Runs
on a single-GPU box, where the torchrun-based multi-GPU tests skip."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import cannikin_synth as synth  # noqa: E402
import paper_2402_05302_b200 as ck  # noqa: E402
from oracle import aggregate as agg  # noqa: E402
from paper_2402_05302_b200 import torch_api as ta  # noqa: E402

import parity  # noqa: E402

TOL = {"f32": 1e-5, "bf16": 1e-2}
TDT = {"f32": torch.float32, "bf16": torch.bfloat16}
KNOBS = ("CANNIKIN_AR_DYN", "CANNIKIN_AR_PUSH", "CANNIKIN_AR_LL", "CANNIKIN_AR_LL128")
VARIANTS = {  # CANNIKIN_AR_DYN, _PUSH, _LL, _LL128 (None: automatic choice by size)
    "static": ("0", "0", "0", "0"), "dyn": ("1", "0", "0", "0"), "push": ("0", "1", "0", "0"),
    "ll": ("0", "0", "1", "0"), "ll128": ("0", "0", "0", "1"), "auto": None,
}
CASES = [(1, "f32", 1), (7, "bf16", 2), (4099, "f32", 3), (300_001, "f32", 4),
         ((1 << 20) + 5, "bf16", 5), (3_000_011, "f32", 6)]


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def _group(world, variant, check_ratios=False, heap_bytes=16 << 20, extra_env=None):
    env = dict(CANNIKIN_SPIN_TIMEOUT_MS="20000", **(extra_env or {}))
    if VARIANTS[variant] is not None:
        env.update(zip(KNOBS, VARIANTS[variant]))
    os.environ.update(env)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    grid = min(32, sms // world)  # W = 8: 18 CTAs per rank, 144 co-resident
    try:
        return ck.Context.group_local(world, device=0, heap_bytes=heap_bytes, grid=grid,
                                      check_ratios=check_ratios)
    finally:
        for k in env:
            if k != "CANNIKIN_SPIN_TIMEOUT_MS":
                os.environ.pop(k, None)


def _reduce(ctxs, tensors, r, streams=None):
    """All ranks' reductions as ONE group launch (cannikin_weighted_allreduce_group); with
    `streams`, instead one per-rank call per stream, issued concurrently."""
    torch.cuda.synchronize()
    if streams is None:
        ta.weighted_allreduce_group(ctxs, tensors, r)
    else:
        for c, t, ri, s in zip(ctxs, tensors, r, streams):
            ta.weighted_allreduce(c, t, ri, stream=s)
    torch.cuda.synchronize()


def _stats(ctxs, streams=None):
    if streams is None:
        return [c.gns_stats() for c in ctxs]
    return [c.gns_stats(stream=s) for c, s in zip(ctxs, streams)]


@pytest.mark.parametrize("world", [2, 3, 4, 8])
@pytest.mark.parametrize("variant", list(VARIANTS))
def test_group_local_parity(world, variant):
    _need_gpu()
    ctxs = _group(world, variant)
    try:
        for N, dtype, seed in CASES:
            b = [int(x) for x in np.random.default_rng(seed).integers(1, 97, size=world)]
            gs = synth.gns_gradients(world, N, b, seed=seed, dtype=dtype)
            r = agg.ratios(b)
            g_ref, ls_ref, gsq_ref = agg.aggregate(gs, r, dtype)
            scale = np.maximum(agg.elementwise_scale([agg.to_f64(g, dtype) for g in gs], r), 1e-30)
            for staged in (False, True):
                if staged:
                    ts = [_to_dev(gs[k], dtype) for k in range(world)]
                else:
                    ts = [ta.bucket_tensor(ctxs[k], N, TDT[dtype]) for k in range(world)]
                    for k in range(world):
                        ts[k].copy_(_to_dev(gs[k], dtype))
                _reduce(ctxs, ts, r)
                outs = [_from_dev(t, dtype) for t in ts]
                st = _stats(ctxs)
                got = agg.to_f64(outs[0], dtype)
                assert np.max(np.abs(got - g_ref) / scale) <= TOL[dtype], (variant, N, staged)
                for k in range(1, world):
                    assert np.array_equal(outs[k], outs[0]), (variant, N, k)
                    assert st[k][0] == st[0][0] and st[k][1] == st[0][1], (variant, N, k)
                assert np.allclose(st[0][0], ls_ref, rtol=1e-4, atol=0), (variant, N)
                assert abs(st[0][1] - gsq_ref) <= 1e-4 * max(gsq_ref, 1e-300), (variant, N)
                if not staged:
                    for k in range(world):
                        ta.free_bucket_tensor(ctxs[k], ts[k])
    finally:
        for c in ctxs:
            c.close()


def test_group_local_bits_identical_across_variants():
    _need_gpu()
    world = 2
    results = {}
    for variant in VARIANTS:
        ctxs = _group(world, variant)
        try:
            for N, dtype, seed in ((100_003, "f32", 21), (200_011, "bf16", 22)):
                b = [5, 17]
                gs = synth.gns_gradients(world, N, b, seed=seed, dtype=dtype)
                ts = [_to_dev(gs[k], dtype) for k in range(world)]
                _reduce(ctxs, ts, agg.ratios(b))
                _stats(ctxs)
                results.setdefault((N, dtype), {})[variant] = _from_dev(ts[0], dtype)
        finally:
            for c in ctxs:
                c.close()
    for key, per in results.items():
        ref = per["static"]
        for variant, out in per.items():
            assert np.array_equal(out, ref), (key, variant)


@pytest.mark.parametrize("variant", ["static", "ll", "ll128", "auto"])
@pytest.mark.parametrize("world", [2, 4])
def test_group_local_back_to_back(world, variant):
    """40 calls of mixed sizes and dtypes enqueued back to back (no host sync in between), each on
    its own bucket: the epoch/parity buffer reuse of the flag protocols under pipelining."""
    _need_gpu()
    ctxs = _group(world, variant)
    rng = np.random.default_rng(7)
    try:
        calls = []
        for t in range(40):
            N = int(rng.choice([1, 33, 4099, 65_537, 300_001, 1_000_003]))
            dtype = "bf16" if t % 3 == 1 else "f32"
            b = [int(x) for x in rng.integers(1, 97, size=world)]
            gs = synth.gns_gradients(world, N, b, seed=1000 + t, dtype=dtype)
            calls.append((N, dtype, b, gs, [_to_dev(gs[k], dtype) for k in range(world)]))
        torch.cuda.synchronize()
        for N, dtype, b, gs, ts in calls:
            ta.weighted_allreduce_group(ctxs, ts, agg.ratios(b))
        torch.cuda.synchronize()
        for N, dtype, b, gs, ts in calls:
            r = agg.ratios(b)
            g_ref, _, _ = agg.aggregate(gs, r, dtype)
            scale = np.maximum(agg.elementwise_scale([agg.to_f64(g, dtype) for g in gs], r), 1e-30)
            outs = [_from_dev(t, dtype) for t in ts]
            assert np.max(np.abs(agg.to_f64(outs[0], dtype) - g_ref) / scale) <= TOL[dtype], (N, dtype)
            for k in range(1, world):
                assert np.array_equal(outs[k], outs[0]), (N, dtype, k)
        st = _stats(ctxs)
        for k in range(1, world):
            assert st[k] == st[0]
    finally:
        for c in ctxs:
            c.close()


def test_group_local_check_ratios():
    _need_gpu()
    world = 2
    for variant in ("static", "ll", "ll128"):
        ctxs = _group(world, variant, check_ratios=True)
        try:
            for scale, want in ((1.0, None), (0.9, "DOMAIN"), (1.0, None)):
                ts = [torch.ones(4099, device="cuda") for _ in range(world)]
                _reduce(ctxs, ts, [scale / world] * world)
                for c in ctxs:
                    if want is None:
                        c.gns_stats()
                    else:
                        with pytest.raises(ck.CannikinError) as e:
                            c.gns_stats()
                        assert e.value.name == want
        finally:
            for c in ctxs:
                c.close()


def test_group_local_errors():
    _need_gpu()
    with pytest.raises(ck.CannikinError) as e:
        ck.Context.group_local(1, device=0, heap_bytes=1 << 20, grid=8)
    assert e.value.name == "INVALID"
    with pytest.raises(ck.CannikinError) as e:
        ck.Context.group_local(2, device=0, heap_bytes=1 << 20, grid=0)
    assert e.value.name == "INVALID"
    ctxs = ck.Context.group_local(2, device=0, heap_bytes=1 << 20, grid=8)
    try:
        with pytest.raises(ck.CannikinError) as e:
            ta.ddp_allreduce_mean(ctxs[0], torch.ones(8, device="cuda"))
        assert e.value.name == "UNSUPPORTED"
    finally:
        for c in ctxs:
            c.close()


def _to_dev(a, dtype):
    if dtype == "bf16":
        return torch.from_numpy(a.view(np.int16).copy()).cuda().view(torch.bfloat16)
    return torch.from_numpy(a.copy()).cuda()


def _from_dev(t, dtype):
    if dtype == "bf16":
        return t.view(torch.int16).cpu().numpy().view(np.uint16)
    return t.cpu().numpy()


def test_group_local_config2_eight_ranks():
    """configs[2]'s ResNet-50 gradient (25,557,032 fp32) at its 8 ranks, automatic variant, one
    bucket per rank: the oracle over the whole vectors, identical bits and statistics."""
    _need_gpu()
    world, N = 8, 25_557_032
    os.environ["CANNIKIN_SPIN_TIMEOUT_MS"] = "20000"
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    ctxs = ck.Context.group_local(world, device=0, heap_bytes=N * 4 + 4096, grid=sms // world)
    try:
        b = [21, 8, 5, 21, 8, 5, 20, 8]  # the emulated A100/V100/P100 mix's split at B = 96
        gs = synth.gns_gradients(world, N, b, seed=31, dtype="f32")
        r = agg.ratios(b)
        ts = [ta.bucket_tensor(ctxs[k], N, torch.float32) for k in range(world)]
        for k in range(world):
            ts[k].copy_(_to_dev(gs[k], "f32"))
        _reduce(ctxs, ts, r)
        st = _stats(ctxs)
        outs = [_from_dev(t, "f32") for t in ts]
        g_ref, ls_ref, gsq_ref = agg.aggregate(gs, r, "f32")
        scale = np.maximum(agg.elementwise_scale([agg.to_f64(g, "f32") for g in gs], r), 1e-30)
        assert np.max(np.abs(outs[0].astype(np.float64) - g_ref) / scale) <= 1e-5
        for k in range(1, world):
            assert np.array_equal(outs[k], outs[0]) and st[k] == st[0]
        assert np.allclose(st[0][0], ls_ref, rtol=1e-4, atol=0)
        assert abs(st[0][1] - gsq_ref) <= 1e-4 * gsq_ref
    finally:
        for c in ctxs:
            c.close()


def test_group_local_config3_eight_ranks_full_size():
    """configs[3] at full size (110M bf16, one 220 MB bucket per rank) at 8 ranks: the automatic
    variant is the push two-shot (W >= 4, >= 128 MiB) -- the path an 8-GPU bench takes.  EVERY
    element against the oracle (chunked), norms against the oracle over the whole vectors."""
    _need_gpu()
    world, N = 8, 110_000_000
    os.environ["CANNIKIN_SPIN_TIMEOUT_MS"] = "20000"
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    ctxs = ck.Context.group_local(world, device=0, heap_bytes=N * 2 + 4096, grid=sms // world)
    try:
        b = [21, 8, 5, 21, 8, 5, 20, 8]
        r = agg.ratios(b)
        gs = synth.device_gns_gradients(world, N, b, seed=9, dtype="bf16")
        ts = [ta.bucket_tensor(ctxs[k], N, torch.bfloat16) for k in range(world)]
        for k in range(world):
            ts[k].copy_(gs[k])
        _reduce(ctxs, ts, r)
        st = _stats(ctxs)
        # every element of every rank's result: rank 0's against the oracle, the others bitwise
        _, lsum, gsum = parity.compare_full(ts, gs, r, "bf16", 1e-2, chunk=10_000_000)
        for k in range(1, world):
            assert st[k] == st[0]
        assert np.allclose(st[0][0], lsum, rtol=1e-4, atol=0)
        assert abs(st[0][1] - gsum) <= 1e-4 * gsum
    finally:
        for c in ctxs:
            c.close()


def test_group_local_ll128_size_limit():
    """The LL128 kernel at its buffer limit (CANNIKIN_LL128_MAX_MB=64: 16,777,216 fp32 elements)
    and 4 KiB past it (the two-shot takes over through the staging copy), W = 2: parity with the
    oracle and identical bits on both ranks on either side of the boundary."""
    _need_gpu()
    world = 2
    ctxs = _group(world, "ll128", heap_bytes=(64 << 20) + 4096,
                  extra_env={"CANNIKIN_LL128_MAX_MB": "64"})
    try:
        for N in ((64 << 20) // 4, (64 << 20) // 4 + 1024):
            b = [37, 91]
            gs = synth.gns_gradients(world, N, b, seed=N % 1000, dtype="f32")
            r = agg.ratios(b)
            ts = [_to_dev(gs[k], "f32") for k in range(world)]
            _reduce(ctxs, ts, r)
            st = _stats(ctxs)
            outs = [_from_dev(t, "f32") for t in ts]
            g_ref, ls_ref, gsq_ref = agg.aggregate(gs, r, "f32")
            scale = np.maximum(agg.elementwise_scale([agg.to_f64(g, "f32") for g in gs], r), 1e-30)
            assert np.max(np.abs(outs[0].astype(np.float64) - g_ref) / scale) <= 1e-5, N
            assert np.array_equal(outs[0], outs[1]) and st[0] == st[1], N
            assert np.allclose(st[0][0], ls_ref, rtol=1e-4, atol=0), N
            assert abs(st[0][1] - gsq_ref) <= 1e-4 * gsq_ref, N
    finally:
        for c in ctxs:
            c.close()


@pytest.mark.parametrize("variant", ["static", "ll", "ll128", "auto"])
def test_group_local_concurrent_streams_match_group_launch(variant):
    """The multi-process call pattern on one GPU: every rank's own cannikin_weighted_allreduce on
    its own stream, issued concurrently (grid * W <= SMs keeps the W kernels co-resident).  The
    result bits and statistics equal the single-launch group call's, and the oracle's values."""
    _need_gpu()
    world = 2
    ctxs = _group(world, variant)
    try:
        for N, dtype, seed in ((4099, "f32", 31), (1_000_003, "bf16", 32), (3_000_011, "f32", 33)):
            b = [11, 29]
            r = agg.ratios(b)
            gs = synth.gns_gradients(world, N, b, seed=seed, dtype=dtype)
            a = [_to_dev(gs[k], dtype) for k in range(world)]
            _reduce(ctxs, a, r)
            st_a = _stats(ctxs)
            streams = [torch.cuda.Stream() for _ in range(world)]
            c = [_to_dev(gs[k], dtype) for k in range(world)]
            _reduce(ctxs, c, r, streams)
            st_c = _stats(ctxs, streams)
            for k in range(world):
                assert np.array_equal(_from_dev(a[k], dtype), _from_dev(c[k], dtype)), (N, k)
                assert st_a[k] == st_c[k]
            g_ref, ls_ref, gsq_ref = agg.aggregate(gs, r, dtype)
            scale = np.maximum(agg.elementwise_scale([agg.to_f64(g, dtype) for g in gs], r), 1e-30)
            got = agg.to_f64(_from_dev(c[0], dtype), dtype)
            assert np.max(np.abs(got - g_ref) / scale) <= TOL[dtype]
            assert np.allclose(st_c[0][0], ls_ref, rtol=1e-4, atol=0)
    finally:
        for cc in ctxs:
            cc.close()


def test_group_launch_errors():
    _need_gpu()
    ctxs = ck.Context.group_local(2, device=0, heap_bytes=1 << 20, grid=8)
    other = ck.Context.group_local(2, device=0, heap_bytes=1 << 20, grid=8)
    x = [torch.ones(1024, device="cuda") for _ in range(2)]
    try:
        for bad in ([ctxs[1], ctxs[0]], [ctxs[0], other[1]]):  # rank order; one group
            with pytest.raises(ck.CannikinError) as e:
                ta.weighted_allreduce_group(bad, x, [0.5, 0.5])
            assert e.value.name == "INVALID"
        with pytest.raises(ck.CannikinError) as e:
            ta.weighted_allreduce_group(ctxs, x, [0.5, float("nan")])
        assert e.value.name == "DOMAIN"
        y = [torch.ones(1025, device="cuda")[1:] for _ in range(2)]  # 4-byte offset: misaligned
        with pytest.raises(ck.CannikinError) as e:
            ta.weighted_allreduce_group(ctxs, y, [0.5, 0.5])
        assert e.value.name == "INVALID"
    finally:
        for c in ctxs + other:
            c.close()
