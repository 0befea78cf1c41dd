#!/usr/bin/env python
"""Bucket-size sweep of the NVLink weighted all-reduce (K3) against NCCL (BASELINE configs[4]:
355M-parameter gradient, buckets 1 MB - 1 GB, equal-split DDP baseline = ncclAllReduce(avg)).

    torchrun --nproc-per-node N tools/k3_sweep.py [--dtype f32|bf16] [--grids 148]

Per bucket size: the gradient (355M elements) is cut into buckets of that size; one "step" = all
buckets reduced back to back (graph-captured, events around the step); busbw = (N s / t) 2(n-1)/n
per rank; max over ranks.  Rank 0 prints JSON lines.
"""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cannikin_synth as synth  # noqa: E402
from paper_2402_05302_b200 import torch_api as ta  # noqa: E402

TOTAL = 354_823_168


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    e0 = torch.cuda.Event(enable_timing=True, external=True)
    e1 = torch.cuda.Event(enable_timing=True, external=True)
    with torch.cuda.graph(g):
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
    g.replay()
    torch.cuda.synchronize()
    dist.barrier()
    g.replay()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / reps], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def main():
    os.environ.setdefault("CANNIKIN_SPIN_TIMEOUT_MS", "120000")  # report, do not hang
    ap = argparse.ArgumentParser()
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--grids", default="0")
    ap.add_argument("--variants", default="0",
                    help="CANNIKIN_AR_DYN values (two-shot), 'push', 'll', 'll128', 'k4' (NCCL path) or 'auto'")
    ap.add_argument("--sizes-mb", default="1,4,16,64,256,1024")
    ap.add_argument("--total", type=int, default=TOTAL)
    ap.add_argument("--nvls", action="store_true", help="also time the NVLS kernel (fp32)")
    ap.add_argument("--gated", default="0", help="0, 1 or 0,1: CANNIKIN_INIT_GATED_ENTRY")
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    lr = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(lr)
    dist.init_process_group("nccl", device_id=torch.device("cuda", lr))
    tdt = {"f32": torch.float32, "bf16": torch.bfloat16}[args.dtype]
    s = 4 if args.dtype == "f32" else 2
    N = args.total
    b = list(range(1, world + 1))
    r = b[rank] / sum(b)
    combos = [(int(g), v, int(gt)) for g in args.grids.split(",") for v in args.variants.split(",")
              for gt in args.gated.split(",")]
    for grid, var, gated in combos:
        knobs = ("CANNIKIN_AR_PUSH", "CANNIKIN_AR_DYN", "CANNIKIN_AR_LL", "CANNIKIN_AR_LL128")
        if var == "auto":
            for k in knobs:
                os.environ.pop(k, None)
        else:
            os.environ.update(dict.fromkeys(knobs, "0"))
            if var == "ll":
                os.environ["CANNIKIN_AR_LL"] = "1"
            elif var == "ll128":
                os.environ["CANNIKIN_AR_LL128"] = "1"
            elif var == "push":
                os.environ["CANNIKIN_AR_PUSH"] = "1"
            elif var != "k4":
                os.environ["CANNIKIN_AR_DYN"] = var
        ctx = ta.init_distributed_context(heap_bytes=N * s, grid=grid, gated=bool(gated))
        bucket = ta.bucket_tensor(ctx, N, tdt)
        mcb = ta.McBucket(N, tdt) if args.nvls else None
        if mcb is not None:
            mcb.tensor.normal_()
        bucket.copy_(synth.device_gns_gradients(world, N, b, seed=0, dtype=args.dtype,
                                                ranks=[rank])[0])
        for mb in [float(x) for x in args.sizes_mb.split(",")]:
            be = max(8, int(mb * 2**20) // s)
            be -= be % 8
            cuts = list(range(0, N, be)) + [N]
            nb = len(cuts) - 1
            reps = max(1, min(20, int(2e9 // (N * s)), 4096 // nb))

            AR = ta.weighted_allreduce_nccl if var == "k4" else ta.weighted_allreduce

            def ours():
                for a, c in zip(cuts[:-1], cuts[1:]):
                    AR(ctx, bucket[a:c], r)
                ctx.gns_stats_async(stats.data_ptr(), torch.cuda.current_stream())

            def nccl():
                for a, c in zip(cuts[:-1], cuts[1:]):
                    ta.ddp_allreduce_mean(ctx, bucket[a:c])

            stats = torch.zeros(world + 1, dtype=torch.float64, device="cuda")
            t_ours = timed(ours, reps)
            t_nccl = timed(nccl, reps)
            t_nvls = None
            if args.nvls and args.dtype == "f32":
                def nvls():
                    for a, c in zip(cuts[:-1], cuts[1:]):
                        ta.weighted_allreduce_nvls(ctx, mcb, r, view=mcb.tensor[a:c])
                    ctx.gns_stats_async(stats.data_ptr(), torch.cuda.current_stream())
                t_nvls = timed(nvls, reps)
            bus = lambda t: N * s / (t * 1e-3) * 2 * (world - 1) / world / 1e9  # noqa: E731
            if rank == 0:
                print(json.dumps({"world": world, "dtype": args.dtype, "grid": grid, "variant": var,
                                  "gated": bool(gated),
                                  "bucket_MB": mb, "buckets": nb, "total_MB": round(N * s / 2**20),
                                  "ours_ms": round(t_ours, 4), "nccl_ms": round(t_nccl, 4),
                                  "ours_busbw": round(bus(t_ours), 1),
                                  "nccl_busbw": round(bus(t_nccl), 1),
                                  "speedup_vs_nccl": round(t_nccl / t_ours, 3),
                                  "nvls_ms": None if t_nvls is None else round(t_nvls, 4),
                                  "nvls_busbw": None if t_nvls is None else round(bus(t_nvls), 1)}),
                      flush=True)
        ta.free_bucket_tensor(ctx, bucket)
        del bucket
        dist.barrier()
        ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
