"""Per-rank worker for tests/test_gpu_multi.py (launched by torchrun, one process per GPU).

Every rank draws ALL ranks' inputs of record on the host from the shared seeded generator (small
sizes), loads its own into a bucket, runs cannikin_weighted_allreduce through the C ABI, and
writes its output bits and norm statistics to <outdir>/rank<r>_<case>.npz for the parent test to
compare against the oracle and across ranks.
"""
import argparse
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import cannikin_synth as synth  # noqa: E402
import paper_2402_05302_b200 as ck  # noqa: E402
from paper_2402_05302_b200 import torch_api as ta  # noqa: E402

CASES = [  # (name, N, dtype, seed)
    ("tiny1", 1, "f32", 1),
    ("odd7", 7, "bf16", 2),
    ("small", 4099, "f32", 3),
    ("mid_f32", (1 << 20) + 3, "f32", 4),
    ("mid_bf16", (1 << 20) + 5, "bf16", 5),
    ("big_bf16", 3_000_011, "bf16", 6),
    ("resnet18", 11_689_512, "f32", 7),    # configs[1]
    ("resnet50", 25_557_032, "f32", 11),   # configs[2]
    ("os_f32", 300_001, "f32", 8),     # LL sized: several CTAs, ragged tail
    ("os_bf16", 600_007, "bf16", 10),
    # multiples of 64 elements: every shard full (the NCCL path's in-place fast paths)
    ("pow2_f32", 1 << 20, "f32", 12),
    ("pow2_bf16", 1 << 21, "bf16", 13),
]


MIXED_CALLS = 40


def b_for(world, seed):
    rng = np.random.default_rng(100 + seed)
    return [int(x) for x in rng.integers(1, 97, size=world)]


def to_dev(a, dtype):
    if dtype == "bf16":
        return torch.from_numpy(a.view(np.int16).copy()).cuda().view(torch.bfloat16)
    return torch.from_numpy(a.copy()).cuda()


def from_dev(t, dtype):
    if dtype == "bf16":
        return t.view(torch.int16).cpu().numpy().view(np.uint16)
    return t.cpu().numpy()


FULL = {  # BASELINE configs at full size in the bench launch configurations: (N, dtype, seed, MB)
    "c4": (110_000_000, "bf16", 9, 0),
    "c5": (354_823_168, "f32", 19, 0),
    "c4b25": (110_000_000, "bf16", 9, 25),  # the bench's bucketed_25mb sidecar: 9 calls (LL128)
}


def full_case(ctx, rank, world, out, cfg):
    """One BASELINE config at full size in the bench launch configuration (one zero-copy bucket,
    default grid).  Every rank's input of record and result are gathered to rank 0 (plumbing),
    which compares EVERY element of rank 0's result with the oracle chunk by chunk and every other
    rank's result bitwise with rank 0's (tests/parity.py), and saves the oracle's whole-vector
    norms; every rank saves its statistics."""
    import parity

    N, dt, seed, bucket_mb = FULL[cfg]
    tdt = torch.bfloat16 if dt == "bf16" else torch.float32
    b = b_for(world, seed)
    B = sum(b)
    g = synth.device_gns_gradients(world, N, b, seed=seed, dtype=dt, ranks=[rank])[0]
    bucket = ta.bucket_tensor(ctx, N, tdt)
    bucket.copy_(g)
    ins = [torch.empty_like(g) for _ in range(world)]
    dist.all_gather(ins, g)  # plumbing: every rank's input of record, for the oracle on rank 0
    del g
    if bucket_mb == 0:
        ta.weighted_allreduce(ctx, bucket, b[rank] / B)
    else:
        be = int(bucket_mb * 2**20) // (2 if dt == "bf16" else 4)
        be -= be % 8
        cuts = list(range(0, N, be)) + [N]
        for a, c in zip(cuts[:-1], cuts[1:]):
            ta.weighted_allreduce(ctx, bucket[a:c], b[rank] / B)
    loc, glob = ctx.gns_stats()
    outs = [torch.empty_like(bucket) for _ in range(world)]
    dist.all_gather(outs, bucket)
    res = {"loc": np.array(loc), "glob": glob, "b": np.array(b)}
    if rank == 0:
        from oracle import aggregate as agg
        err, lsum, gsum = parity.compare_full(outs, ins, agg.ratios(b), dt,
                                              1e-2 if dt == "bf16" else 1e-5, chunk=20_000_000)
        res.update(max_err=err, oracle_loc=lsum, oracle_glob=gsum)
    np.savez(os.path.join(out, f"rank{rank}_full.npz"), **res)
    ta.free_bucket_tensor(ctx, bucket)
    del ins, outs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--grid", type=int, default=0)
    ap.add_argument("--full", default="", choices=["", "c4", "c5", "c4b25"])
    ap.add_argument("--variants", action="store_true")
    ap.add_argument("--mixed", action="store_true")
    ap.add_argument("--gated", action="store_true",
                    help="with --mixed: CANNIKIN_INIT_GATED_ENTRY, and one rank arrives late "
                         "(a 2 ms device busy-wait before its call) at every call")
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    lr = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(lr)
    dist.init_process_group("nccl", device_id=torch.device("cuda", lr))
    maxN = max(c[1] for c in CASES)
    if args.mixed:
        # a seeded random sequence of sizes, dtypes and buffer kinds under the automatic variant
        # choice: LL, two-shot pull/dynamic/push and staged calls interleave on one ctx, so the
        # epochs, parities and statistics rows of the different kernels must compose
        ctx = ta.init_distributed_context(heap_bytes=(24 << 20), grid=args.grid, gated=args.gated)
        rng = np.random.default_rng(77)
        tdt = {"f32": torch.float32, "bf16": torch.bfloat16}
        for t in range(MIXED_CALLS):
            N = int(rng.choice([1, 3, 1000, 4099, 65_537, 300_001, 1_000_003, 2_500_001, 5_000_011]))
            dtype = "f32" if rng.random() < 0.5 else "bf16"
            staged = bool(rng.random() < 0.3)
            b = b_for(world, 200 + t)
            gs = synth.gns_gradients(world, N, b, seed=200 + t, dtype=dtype)
            if staged:
                x = to_dev(gs[rank], dtype)
            else:
                x = ta.bucket_tensor(ctx, N, tdt[dtype])
                x.copy_(to_dev(gs[rank], dtype))
            torch.cuda.synchronize()
            if args.gated and rank == t % world:
                ck.emulate_compute(2e-3, torch.cuda.current_stream().cuda_stream)  # late rank
            ta.weighted_allreduce(ctx, x, b[rank] / sum(b))
            launches = ctx.last_launch_count()
            loc, glob = ctx.gns_stats()
            np.savez(os.path.join(args.out, f"rank{rank}_mixed_{t}.npz"), out=from_dev(x, dtype),
                     loc=np.array(loc), glob=glob, N=N, dtype=dtype, b=np.array(b),
                     launches=launches, staged=staged)
            if not staged:
                ta.free_bucket_tensor(ctx, x)
        # the same ctx inside a CUDA graph: [fill, reduce] (gate + reduction kernel when gated)
        # captured once, replayed three times with a late rank each time; the epochs live on the
        # device, so every replay is a fresh, correct reduction (LL, LL128 and two-shot sizes)
        graph_ok = []
        for Ng in (1000, 300_001, 5_000_011):
            x = ta.bucket_tensor(ctx, Ng, torch.float32)
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                x.fill_(float(rank + 1))
                ta.weighted_allreduce(ctx, x, 1.0 / world)
            for rep in range(3):
                dist.barrier()
                if args.gated and rank == rep % world:
                    ck.emulate_compute(2e-3, torch.cuda.current_stream().cuda_stream)
                g.replay()
                torch.cuda.synchronize()
                graph_ok.append(bool(torch.allclose(x, torch.full_like(x, (world + 1) / 2))))
            ctx.gns_stats()
            del g
            ta.free_bucket_tensor(ctx, x)
        np.save(os.path.join(args.out, f"rank{rank}_graph_replays.npy"), np.array(graph_ok))
        dist.barrier()
        ctx.close()
        dist.destroy_process_group()
        return
    if args.variants:
        # the same inputs through every K3 variant: the result bits must not depend on it
        VARS = {"static": ("0", "0", "0", "0"), "dyn": ("1", "0", "0", "0"),
                "push": ("0", "1", "0", "0"), "ll": ("0", "0", "1", "0"),
                "ll128": ("0", "0", "0", "1")}
        for name, (dyn, push, ll, ll128) in VARS.items():
            os.environ.update(CANNIKIN_AR_DYN=dyn, CANNIKIN_AR_PUSH=push, CANNIKIN_AR_LL=ll,
                              CANNIKIN_AR_LL128=ll128)
            ctx = ta.init_distributed_context(heap_bytes=(1 << 22), grid=args.grid)
            for N, dtype in ((100_003, "f32"), (200_011, "bf16")):
                b = b_for(world, 21)
                gs = synth.gns_gradients(world, N, b, seed=21, dtype=dtype)
                t = ta.bucket_tensor(ctx, N, {"f32": torch.float32, "bf16": torch.bfloat16}[dtype])
                t.copy_(to_dev(gs[rank], dtype))
                ta.weighted_allreduce(ctx, t, b[rank] / sum(b))
                ctx.gns_stats()
                np.save(os.path.join(args.out, f"rank{rank}_var_{name}_{dtype}.npy"), from_dev(t, dtype))
                ta.free_bucket_tensor(ctx, t)
            dist.barrier()
            ctx.close()
        dist.destroy_process_group()
        return
    if args.full:
        N, dt, _, _ = FULL[args.full]
        ctx = ta.init_distributed_context(heap_bytes=N * (2 if dt == "bf16" else 4) + 4096,
                                          grid=args.grid)
        full_case(ctx, rank, world, args.out, args.full)
        dist.barrier()
        ctx.close()
        dist.destroy_process_group()
        return
    ctx = ta.init_distributed_context(heap_bytes=maxN * 4 + 4096, grid=args.grid)
    # CANNIKIN_TEST_PATH=nccl: the cases go through the NCCL path (K4) instead of the P2P kernels
    AR = ta.weighted_allreduce_nccl if os.environ.get("CANNIKIN_TEST_PATH") == "nccl" else ta.weighted_allreduce
    tdt = {"f32": torch.float32, "bf16": torch.bfloat16}
    for name, N, dtype, seed in CASES:
        b = b_for(world, seed)
        B = sum(b)
        gs = synth.gns_gradients(world, N, b, seed=seed, dtype=dtype)
        # (1) zero-copy bucket in the symmetric heap
        bucket = ta.bucket_tensor(ctx, N, tdt[dtype])
        bucket.copy_(to_dev(gs[rank], dtype))
        AR(ctx, bucket, b[rank] / B)
        # (5) out-of-place statistics of the unreduced gradient (cannikin_gns_stats_bucket), while
        # (1)'s fused statistics are pending: the bucket is not modified and (1)'s are kept
        src = to_dev(gs[rank], dtype)
        loc5, glob5 = ta.gns_stats_bucket(ctx, src, b[rank])
        same5 = bool(torch.equal(src.view(torch.int16) if dtype == "bf16" else src,
                                 to_dev(gs[rank], dtype).view(torch.int16) if dtype == "bf16"
                                 else to_dev(gs[rank], dtype)))
        loc, glob = ctx.gns_stats()
        out1 = from_dev(bucket, dtype)
        # (2) again (determinism, flag epochs advance)
        bucket.copy_(to_dev(gs[rank], dtype))
        AR(ctx, bucket, b[rank] / B)
        loc2, glob2 = ctx.gns_stats()
        out2 = from_dev(bucket, dtype)
        ta.free_bucket_tensor(ctx, bucket)
        # (3) ordinary (non-peer-mapped) torch tensor: staged through the heap scratch
        t = to_dev(gs[rank], dtype)
        AR(ctx, t, b[rank] / B)
        loc3, glob3 = ctx.gns_stats()
        out3 = from_dev(t, dtype)
        # (4) the same gradient as 3 buckets of different sizes; stats accumulate over buckets
        t = to_dev(gs[rank], dtype)
        cuts = sorted({0, N // 3 - (N // 3) % 8, (2 * N) // 3 - ((2 * N) // 3) % 8, N})
        for a, c in zip(cuts[:-1], cuts[1:]):
            AR(ctx, t[a:c], b[rank] / B)
        loc4, glob4 = ctx.gns_stats()
        out4 = from_dev(t, dtype)
        np.savez(os.path.join(args.out, f"rank{rank}_{name}.npz"), out1=out1, out2=out2,
                 out3=out3, out4=out4, loc=np.array(loc), glob=glob, loc2=np.array(loc2),
                 glob2=glob2, loc3=np.array(loc3), glob3=glob3, loc4=np.array(loc4), glob4=glob4,
                 loc5=np.array(loc5), glob5=glob5, same5=same5, b=np.array(b))
    # guard bands: buckets A | B | C adjacent in the heap; reducing B (ragged) must not touch A, C
    for N in (1, 7, 4099, (1 << 20) + 3):
        for dtype in ("f32", "bf16"):
            A = ta.bucket_tensor(ctx, 4096, tdt[dtype])
            Bk = ta.bucket_tensor(ctx, N, tdt[dtype])
            C = ta.bucket_tensor(ctx, 4096, tdt[dtype])
            A.fill_(-3.0)
            C.fill_(-3.0)
            Bk.copy_(to_dev(synth.gns_gradients(world, N, [1] * world, seed=N)[rank], "f32").to(tdt[dtype]))
            ta.weighted_allreduce(ctx, Bk, 1.0 / world)
            torch.cuda.synchronize()
            ok = bool(torch.all(A == -3.0)) and bool(torch.all(C == -3.0))
            np.save(os.path.join(args.out, f"rank{rank}_canary_{dtype}_{N}.npy"), np.array([ok]))
            ta.free_bucket_tensor(ctx, C)
            ta.free_bucket_tensor(ctx, Bk)
            ta.free_bucket_tensor(ctx, A)
    ctx.gns_stats()
    # CANNIKIN_INIT_CHECK_RATIOS: shares summing to 1 pass; shares summing to 0.95 are reported as
    # DOMAIN (the reduction itself still runs) and the condition is cleared by the report
    ctx2 = ta.init_distributed_context(heap_bytes=1 << 20, grid=args.grid, check_ratios=True)
    chk = {}
    for tag, scale in (("ok", 1.0), ("bad", 0.95), ("ok_after", 1.0)):
        t = ta.bucket_tensor(ctx2, 4099, torch.float32)
        t.fill_(1.0)
        AR(ctx2, t, scale / world)  # the P2P kernels, or K4 under CANNIKIN_TEST_PATH=nccl
        try:
            ctx2.gns_stats()
            chk[tag] = "OK"
        except ck.CannikinError as e:
            chk[tag] = e.name
        chk[tag + "_val"] = float(t[0])
        ta.free_bucket_tensor(ctx2, t)
    np.save(os.path.join(args.out, f"rank{rank}_check_ratios.npy"), np.array([chk["ok"], chk["bad"], chk["ok_after"]]))
    np.save(os.path.join(args.out, f"rank{rank}_check_ratios_val.npy"),
            np.array([chk["ok_val"], chk["bad_val"], chk["ok_after_val"]]))
    dist.barrier()
    ctx2.close()
    # the bench's live NVLink ceiling probe runs (collective) and leaves the ctx usable
    for cps in (1, 2, 4):
        ctx.probe_a2a_write(1 << 20, 3, cps)
    torch.cuda.synchronize()
    dist.barrier()
    t = ta.bucket_tensor(ctx, 4099, torch.float32)
    t.fill_(float(rank + 1))
    ta.weighted_allreduce(ctx, t, 1.0 / world)
    ctx.gns_stats()
    np.save(os.path.join(args.out, f"rank{rank}_probe.npy"), t.cpu().numpy())
    ta.free_bucket_tensor(ctx, t)
    # DDP baseline semantics: mean of the ranks' buffers
    x = torch.full((1000,), float(rank + 1), device="cuda")
    ta.ddp_allreduce_mean(ctx, x)
    torch.cuda.synchronize()
    np.save(os.path.join(args.out, f"rank{rank}_ddp.npy"), x.cpu().numpy())
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
