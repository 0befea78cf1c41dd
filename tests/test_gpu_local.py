"""GPU parity of the single-GPU path (K2 emulated ranks; world-1 weighted_allreduce) against the
oracle, through the C ABI.  Tolerances (BASELINE.json north_star; readings Q1-Q3 of DESIGN.md §4):
  g        : max_e |gpu_e - ref_e| / max(sum_i |r_i g_i[e]|, 1e-30) <= 1e-5 (fp32), 1e-2 (bf16)
  norms    : relative 1e-4
  GNS      : G, S within 1e-4 of the oracle's scale (Q3)
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import cannikin_synth as synth  # noqa: E402
import paper_2402_05302_b200 as ck  # noqa: E402
from paper_2402_05302_b200 import torch_api as ta  # noqa: E402
from oracle import aggregate as agg  # noqa: E402
from oracle import gns as ogns  # noqa: E402

import parity  # noqa: E402

TOL = {"f32": 1e-5, "bf16": 1e-2}
TDT = {"f32": torch.float32, "bf16": torch.bfloat16}


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    c = ck.Context(world=1, device=0)
    yield c
    c.close()


def to_dev(a, dtype):
    if dtype == "bf16":
        return torch.from_numpy(a.view(np.int16).copy()).cuda().view(torch.bfloat16)
    return torch.from_numpy(a.copy()).cuda()


def from_dev(t, dtype):
    if dtype == "bf16":
        return t.view(torch.int16).cpu().numpy().view(np.uint16)
    return t.cpu().numpy()


def run_local(ctx, gs, r, dtype, out=None, accumulate=False, local=None, glob=None, variant=None):
    ins = [to_dev(g, dtype) for g in gs]
    N = ins[0].numel()
    if out is None:
        out = torch.empty(N, dtype=TDT[dtype], device="cuda")
    if local is None:
        local = torch.zeros(len(gs), dtype=torch.float64, device="cuda")
        glob = torch.zeros(1, dtype=torch.float64, device="cuda")
    ta.weighted_sum_local(ctx, ins, r, out, local, glob, accumulate=accumulate, variant=variant)
    torch.cuda.synchronize()
    return out, local, glob, ins


def check(gs, r, dtype, out, local, glob):
    g_ref, ls_ref, gs_ref = agg.aggregate(gs, r, dtype)
    gs64 = [agg.to_f64(g, dtype) for g in gs]
    got = agg.to_f64(from_dev(out, dtype), dtype)
    if got.size:
        scale = np.maximum(agg.elementwise_scale(gs64, r), 1e-30)
        err = np.max(np.abs(got - g_ref) / scale)
        assert err <= TOL[dtype], err
    ls = local.cpu().numpy()
    for j in range(len(gs)):
        assert abs(ls[j] - ls_ref[j]) <= 1e-4 * max(ls_ref[j], 1e-300), (j, ls[j], ls_ref[j])
    gv = float(glob.cpu()[0])
    assert abs(gv - gs_ref) <= 1e-4 * max(gs_ref, 1e-300), (gv, gs_ref)
    return g_ref, ls_ref, gs_ref


@pytest.mark.parametrize("variant", ["ldg", "tma"])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("nr", [1, 2, 3, 5, 8, 16])
@pytest.mark.parametrize("N", [1, 7, 4099, (1 << 20) + 3])
def test_parity_sizes_ranks(ctx, dtype, nr, N, variant):
    b = [int(x) for x in np.random.default_rng(nr * 7 + N).integers(1, 200, size=nr)]
    gs = synth.gns_gradients(nr, N, b, seed=nr + N, dtype=dtype)
    r = agg.ratios(b)
    out, local, glob, _ = run_local(ctx, gs, r, dtype, variant=variant)
    check(gs, r, dtype, out, local, glob)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_variants_identical_output_bits(ctx, dtype):
    b = [7, 1, 30, 12, 5]
    gs = synth.gns_gradients(5, 3_000_017, b, seed=12, dtype=dtype)
    r = agg.ratios(b)
    o1, l1, g1, _ = run_local(ctx, gs, r, dtype, variant="ldg")
    o2, l2, g2, _ = run_local(ctx, gs, r, dtype, variant="tma")
    v = (lambda t: t.view(torch.int16)) if dtype == "bf16" else (lambda t: t)
    assert torch.equal(v(o1), v(o2))
    assert torch.allclose(l1, l2, rtol=1e-12) and torch.allclose(g1, g2, rtol=1e-12)


def test_config1_end_to_end_gns(ctx):
    """configs[0]: 3 emulated ranks, 2^20 fp32, b = {32, 64, 96}; the GNS estimate through the
    library from the GPU norms matches the oracle's from its own norms (reading Q3)."""
    b = [32, 64, 96]
    gs = synth.gns_gradients(3, 1 << 20, b, seed=0, dtype="f32")
    r = agg.ratios(b)
    out, local, glob, _ = run_local(ctx, gs, r, "f32")
    _, ls_ref, gs_ref = check(gs, r, "f32", out, local, glob)
    est = ck.gns_estimate(local.cpu().tolist(), float(glob.cpu()[0]), b)
    ref = ogns.gns_estimate(ls_ref, gs_ref, b)
    B = sum(b)
    for i in range(3):
        scaleG = (B * gs_ref + b[i] * ls_ref[i]) / (B - b[i])
        scaleS = b[i] * B / (B - b[i]) * (ls_ref[i] + gs_ref)
        assert abs(est["Gi"][i] - ref["Gi"][i]) <= 1e-4 * scaleG
        assert abs(est["Si"][i] - ref["Si"][i]) <= 1e-4 * scaleS
    sG = sum(abs(w) * (B * gs_ref + bb * l) / (B - bb) for w, bb, l in zip(ref["wG"], b, ls_ref))
    sS = sum(abs(w) * bb * B / (B - bb) * (l + gs_ref) for w, bb, l in zip(ref["wS"], b, ls_ref))
    assert abs(est["G2"] - ref["G2"]) <= 1e-4 * sG
    assert abs(est["trS"] - ref["trS"]) <= 1e-4 * sS


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_layered_precision_stress(ctx, dtype):
    gs = synth.layered_gradients(4, (1 << 18) + 5, seed=3, dtype=dtype)
    r = agg.ratios([5, 17, 40, 2])
    out, local, glob, _ = run_local(ctx, gs, r, dtype)
    check(gs, r, dtype, out, local, glob)


def test_special_values(ctx):
    N = 10007
    zeros = [np.zeros(N, dtype=np.float32)] * 3
    out, local, glob, _ = run_local(ctx, zeros, [0.2, 0.3, 0.5], "f32")
    assert not out.any() and not local.any() and not glob.any()
    g = synth.gns_gradients(1, N, [4], seed=1)[0]
    out, local, glob, _ = run_local(ctx, [g, g, g], [0.0, 1.0, 0.0], "f32")
    assert np.array_equal(out.cpu().numpy(), g)  # one-hot r copies g_1 exactly
    gs = synth.gns_gradients(3, N, [1, 1, 1], seed=2)
    out, local, glob, _ = run_local(ctx, gs, [1 / 3] * 3, "f32")
    check(gs, [1 / 3] * 3, "f32", out, local, glob)  # equal b: plain mean


def test_empty_bucket(ctx):
    out, local, glob, _ = run_local(ctx, [np.zeros(0, np.float32)] * 2, [0.5, 0.5], "f32")
    assert not local.any() and not glob.any()


@pytest.mark.parametrize("variant", ["ldg", "tma"])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_deterministic_bitwise(ctx, dtype, variant):
    gs = synth.gns_gradients(5, (1 << 20) + 11, [3, 9, 27, 81, 1], seed=9, dtype=dtype)
    r = agg.ratios([3, 9, 27, 81, 1])
    o1, l1, g1, _ = run_local(ctx, gs, r, dtype, variant=variant)
    o2, l2, g2, _ = run_local(ctx, gs, r, dtype, variant=variant)
    assert torch.equal(o1.view(torch.int16) if dtype == "bf16" else o1,
                       o2.view(torch.int16) if dtype == "bf16" else o2)
    assert torch.equal(l1, l2) and torch.equal(g1, g2)


@pytest.mark.parametrize("variant", ["ldg", "tma"])
def test_in_place_and_accumulate(ctx, variant):
    """out may alias an input; ACCUMULATE sums stats over buckets (multi-bucket gradient)."""
    N = 3 * 65536 + 8
    b = [10, 20, 30]
    gs = synth.gns_gradients(3, N, b, seed=4)
    r = agg.ratios(b)
    ins = [to_dev(g, "f32") for g in gs]
    local = torch.zeros(3, dtype=torch.float64, device="cuda")
    glob = torch.zeros(1, dtype=torch.float64, device="cuda")
    cuts = [0, 65536, 2 * 65536 + 4, N]
    for a, c in zip(cuts[:-1], cuts[1:]):
        ta.weighted_sum_local(ctx, [x[a:c] for x in ins], r, ins[0][a:c], local, glob,
                              accumulate=True, variant=variant)
    torch.cuda.synchronize()
    check(gs, r, "f32", ins[0], local, glob)


@pytest.mark.parametrize("variant", ["ldg", "tma"])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_pdl_chained_buckets(ctx, dtype, variant):
    """CANNIKIN_LOCAL_CHAIN (the bucketed bench): buckets after the first are launched as
    programmatic dependents and start reading while the previous bucket finishes; results and the
    accumulated statistics match the oracle, and the bits equal an unchained run."""
    N = 5 * 300_007 + 3
    b = [4, 9, 1, 30]
    gs = synth.gns_gradients(4, N, b, seed=17, dtype=dtype)
    r = agg.ratios(b)
    ins = [to_dev(g, dtype) for g in gs]
    outs = []
    for chain in (True, False):
        out = torch.empty_like(ins[0])
        local = torch.zeros(4, dtype=torch.float64, device="cuda")
        glob = torch.zeros(1, dtype=torch.float64, device="cuda")
        cuts = [0, 300_000, 2 * 300_000 + 8, 3 * 300_000 + 16, 4 * 300_000, N]
        for i, (a, c) in enumerate(zip(cuts[:-1], cuts[1:])):
            ta.weighted_sum_local(ctx, [x[a:c] for x in ins], r, out[a:c], local, glob,
                                  accumulate=i > 0, variant=variant, chain=chain and i > 0)
        torch.cuda.synchronize()
        check(gs, r, dtype, out, local, glob)
        outs.append((out, local.clone(), glob.clone()))
    v = (lambda t: t.view(torch.int16)) if dtype == "bf16" else (lambda t: t)
    assert torch.equal(v(outs[0][0]), v(outs[1][0]))
    assert torch.equal(outs[0][1], outs[1][1]) and torch.equal(outs[0][2], outs[1][2])


def test_world1_allreduce_and_stats(ctx):
    N = 123457
    g = synth.gns_gradients(1, N, [8], seed=6)[0]
    t = to_dev(g, "f32")
    ta.weighted_allreduce(ctx, t, 1.0)
    loc, glob = ctx.gns_stats()
    ref = agg.sq_norm(agg.to_f64(g, "f32"))
    assert np.array_equal(t.cpu().numpy(), g)
    assert math.isclose(loc[0], ref, rel_tol=1e-6) and math.isclose(glob, ref, rel_tol=1e-6)
    assert ctx.gns_stats() == ([0.0], 0.0)   # reset after read


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_gns_stats_bucket_out_of_place(ctx, dtype):
    """cannikin_gns_stats_bucket (world 1): |g_0|^2 and |g|^2 = |r_0 g_0|^2 with r_0 = b_0/B = 1 of
    an unreduced bucket against the oracle, the bucket unchanged, and the statistics of an earlier
    in-place reduction still pending for gns_stats."""
    N = (3 << 20) + 5
    g = synth.device_gns_gradients(1, N, [12], seed=41, dtype=dtype)[0]
    h = synth.device_gns_gradients(1, N, [12], seed=42, dtype=dtype)[0]
    ref_g = parity.host_bits(g, dtype)
    t = h.clone()
    ta.weighted_allreduce(ctx, t, 1.0)             # fused statistics of h, pending
    loc, glob = ta.gns_stats_bucket(ctx, g, 12)    # out of place, of g
    assert np.array_equal(parity.host_bits(g, dtype), ref_g)
    x = agg.to_f64(ref_g, dtype)
    want = agg.sq_norm(x)
    assert abs(loc[0] - want) <= 1e-4 * want and abs(glob - want) <= 1e-4 * want
    loc_h, glob_h = ctx.gns_stats()
    want_h = agg.sq_norm(agg.to_f64(parity.host_bits(h, dtype), dtype))
    assert abs(loc_h[0] - want_h) <= 1e-4 * want_h and abs(glob_h - want_h) <= 1e-4 * want_h
    with pytest.raises(ck.CannikinError) as e:
        ta.gns_stats_bucket(ctx, g, -1)
    assert e.value.name == "DOMAIN"


def test_errors(ctx):
    x = torch.zeros(1024, device="cuda")
    loc = torch.zeros(17, dtype=torch.float64, device="cuda")
    glob = torch.zeros(1, dtype=torch.float64, device="cuda")
    with pytest.raises(ck.CannikinError) as e:
        ctx.weighted_sum_local([x.data_ptr()] * 17, [1 / 17] * 17, x.data_ptr(), 1024, ck.F32,
                               loc.data_ptr(), glob.data_ptr())
    assert e.value.name == "UNSUPPORTED"
    with pytest.raises(ck.CannikinError) as e:
        ctx.weighted_sum_local([x.data_ptr() + 4], [1.0], x.data_ptr(), 1000, ck.F32,
                               loc.data_ptr(), glob.data_ptr())
    assert e.value.name == "INVALID"
    with pytest.raises(ck.CannikinError) as e:
        ctx.weighted_allreduce(x.data_ptr(), 1024, 7, 1.0)
    assert e.value.name == "UNSUPPORTED"


@pytest.mark.parametrize("variant,bucket_mb", [("ldg", 0), ("tma", 0), ("ldg", 25)])
@pytest.mark.parametrize("nr", [8])
def test_full_size_c4(ctx, nr, variant, bucket_mb):
    """configs[3] at full size in the bench launch configurations: 110M bf16, 8 emulated ranks, as
    one launch and (bench --bucket-mb 25) as 9 PDL-chained 25 MB buckets accumulating the
    statistics.  EVERY element against the oracle (chunked, tests/parity.py); the norms against
    the oracle over the whole vectors."""
    N = 110_000_000
    b = [37, 29, 21, 12, 9, 8, 3, 1]
    gs = synth.device_gns_gradients(nr, N, b, seed=0, dtype="bf16")
    r = agg.ratios(b)
    out = torch.empty(N, dtype=torch.bfloat16, device="cuda")
    local = torch.zeros(nr, dtype=torch.float64, device="cuda")
    glob = torch.zeros(1, dtype=torch.float64, device="cuda")
    if bucket_mb == 0:
        ta.weighted_sum_local(ctx, gs, r, out, local, glob, variant=variant)
    else:
        be = int(bucket_mb * 2**20) // 2
        be -= be % 8
        cuts = list(range(0, N, be)) + [N]
        for i, (a, c) in enumerate(zip(cuts[:-1], cuts[1:])):
            ta.weighted_sum_local(ctx, [g[a:c] for g in gs], r, out[a:c], local, glob,
                                  accumulate=i > 0, chain=i > 0, variant=variant)
    torch.cuda.synchronize()
    _, lsum, gsum = parity.compare_full([out], gs, r, "bf16", TOL["bf16"], chunk=10_000_000)
    assert np.allclose(local.cpu().numpy(), lsum, rtol=1e-4)
    assert abs(float(glob.cpu()[0]) - gsum) <= 1e-4 * gsum


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("nr,N", [(1, (8 << 20) + 3), (2, (8 << 20) + 3), (3, (4 << 20) + 5),
                                  (4, (4 << 20) + 5), (2, 33_554_435)])
def test_unrolled_main_loops_every_element(ctx, dtype, nr, N):
    """The unrolled grid-stride loops of K2 (U = 4 vectors per thread per rank for n <= 2, U = 2 for
    n <= 4; wsum_local.cu) only run once the bucket exceeds (U-1) grid strides (~151k vectors per
    stride at 4 CTAs/SM), i.e. beyond the 2^20-element cases above: 4-33M elements, every element
    against the oracle, both dtypes, ragged tails."""
    b = [int(x) for x in np.random.default_rng(nr + N).integers(1, 100, size=nr)]
    gs = synth.device_gns_gradients(nr, N, b, seed=nr * 3 + 1, dtype=dtype)
    r = agg.ratios(b)
    out = torch.empty(N, dtype=TDT[dtype], device="cuda")
    local = torch.zeros(nr, dtype=torch.float64, device="cuda")
    glob = torch.zeros(1, dtype=torch.float64, device="cuda")
    ta.weighted_sum_local(ctx, gs, r, out, local, glob, variant="ldg")
    torch.cuda.synchronize()
    _, lsum, gsum = parity.compare_full([out], gs, r, dtype, TOL[dtype])
    assert np.allclose(local.cpu().numpy(), lsum, rtol=1e-4)
    assert abs(float(glob.cpu()[0]) - gsum) <= 1e-4 * gsum


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_world1_allreduce_large_every_element(ctx, dtype):
    """world-1 cannikin_weighted_allreduce over a > 8M-element bucket (K2 with n = 1, U = 4 loop):
    g = r_0 g_0 in place, every element against the oracle; statistics through gns_stats."""
    N = (9 << 20) + 7
    g = synth.device_gns_gradients(1, N, [8], seed=21, dtype=dtype)[0]
    t = g.clone()
    ta.weighted_allreduce(ctx, t, 0.625)
    loc, glob = ctx.gns_stats()
    _, lsum, gsum = parity.compare_full([t], [g], [0.625], dtype, TOL[dtype])
    assert abs(loc[0] - lsum[0]) <= 1e-4 * lsum[0]
    assert abs(glob - gsum) <= 1e-4 * gsum


@pytest.mark.parametrize("variant", ["ldg", "tma"])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("N", [1, 7, 9, 4099, 65536 + 3])
def test_no_out_of_bounds_writes(ctx, dtype, N, variant):
    """Guard bands (compute-sanitizer is closed on this pool): inputs and output are slices in the
    middle of canary-filled buffers; every canary byte must survive, ragged tails included."""
    tdt = TDT[dtype]
    pad = 4096
    esz = 4 if dtype == "f32" else 2
    big = [torch.full((N + 2 * pad,), -7.0, dtype=tdt, device="cuda") for _ in range(4)]
    gs = synth.gns_gradients(3, N, [1, 2, 3], seed=N, dtype=dtype)
    for j in range(3):
        big[j][pad:pad + N] = to_dev(gs[j], dtype)
    out_big = big[3]
    stats = torch.full((8,), -5.0, dtype=torch.float64, device="cuda")
    ta.weighted_sum_local(ctx, [b[pad:pad + N] for b in big[:3]], [0.2, 0.3, 0.5],
                          out_big[pad:pad + N], stats[2:5], stats[5:6], variant=variant)
    torch.cuda.synchronize()
    for bb in big:
        assert torch.all(bb[:pad] == -7.0) and torch.all(bb[pad + N:] == -7.0)
    assert torch.all(stats[:2] == -5.0) and torch.all(stats[6:] == -5.0)
    del esz


def test_full_size_c5(ctx):
    """configs[4]'s 355M fp32 gradient at full size on one GPU (3 emulated ranks): EVERY element
    against the oracle (chunked), norms against the oracle over the whole vectors."""
    N, nr = 354_823_168, 3
    b = [5, 17, 40]
    gs = synth.device_gns_gradients(nr, N, b, seed=2, dtype="f32")
    r = agg.ratios(b)
    out = torch.empty(N, dtype=torch.float32, device="cuda")
    local = torch.zeros(nr, dtype=torch.float64, device="cuda")
    glob = torch.zeros(1, dtype=torch.float64, device="cuda")
    ta.weighted_sum_local(ctx, gs, r, out, local, glob)
    torch.cuda.synchronize()
    _, lsum, gsum = parity.compare_full([out], gs, r, "f32", TOL["f32"], chunk=20_000_000)
    assert np.allclose(local.cpu().numpy(), lsum, rtol=1e-4)
    assert abs(float(glob.cpu()[0]) - gsum) <= 1e-4 * gsum


def test_green_partitions_are_disjoint(ctx):
    """cannikin_green_partitions (the bench's shared-GPU heterogeneity harness): kernels launched on
    partition i's stream run only on partition i's SMs, and the partitions do not overlap -- read
    from K2's own per-CTA %smid trace."""
    green = ck.GreenPartitions([16, 8])
    try:
        assert green.sms == [16, 8]
        N = 1 << 22
        gs = synth.gns_gradients(2, N, [3, 5], seed=3)
        ins = [to_dev(g, "f32") for g in gs]
        out = torch.empty(N, device="cuda")
        local = torch.zeros(2, dtype=torch.float64, device="cuda")
        glob = torch.zeros(1, dtype=torch.float64, device="cuda")
        used = []
        for h in green.streams:
            st = torch.cuda.ExternalStream(h)
            st.wait_stream(torch.cuda.current_stream())
            ta.weighted_sum_local(ctx, ins, [0.375, 0.625], out, local, glob, variant="ldg",
                                  stream=st)
            torch.cuda.synchronize()
            check(gs, [0.375, 0.625], "f32", out, local, glob)
            used.append({int(t[1]) for t in ctx.trace()})
        assert 0 < len(used[0]) <= 16 and 0 < len(used[1]) <= 8, used
        assert not (used[0] & used[1]), used
    finally:
        torch.cuda.synchronize()
        green.close()



def test_stream_pattern_probe():
    """cannikin_probe_stream_pattern (the bench's live HBM ceiling for K2): out = word-wise integer
    sum of the inputs, every vector including a ragged grid-stride tail."""
    n = 3 * 65536 + 40  # 32-bit words; a multiple of 4 (16-byte vectors)
    ins = [torch.full((n,), k + 1, dtype=torch.int32, device="cuda") for k in range(5)]
    out = torch.zeros(n, dtype=torch.int32, device="cuda")
    ck.probe_stream_pattern([t.data_ptr() for t in ins], out.data_ptr(), n * 4, 2)
    torch.cuda.synchronize()
    assert torch.all(out == 15)
