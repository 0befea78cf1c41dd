#!/usr/bin/env python
"""Per-phase device timeline of the two-shot kernel (K3) from its built-in %globaltimer trace.
    torchrun --nproc-per-node N tools/k3_trace.py
Prints, per bucket size and rank: event-timed kernel time and the CTA-median / max of
entry-barrier wait, data phase, exit-barrier wait, final reduction (microseconds)."""
import json
import os
import statistics
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_05302_b200 import torch_api as ta  # noqa: E402


def main():
    os.environ.setdefault("CANNIKIN_SPIN_TIMEOUT_MS", "120000")  # report, do not hang
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ.get("LOCAL_RANK", rank))))
    bf16 = "--bf16" in sys.argv
    tdt, es = (torch.bfloat16, 2) if bf16 else (torch.float32, 4)
    sizes = [0.004, 0.0625, 1, 4, 16, 64, 256]
    for a in sys.argv:
        if a.startswith("--sizes="):
            sizes = [float(x) for x in a.split("=", 1)[1].split(",")]
    N = max(64 << 20, int(max(sizes) * 2**20) // es + 64)
    dyn = os.environ.get("CANNIKIN_AR_DYN", "0")
    use_nvls = "--nvls" in sys.argv
    mcb = ta.McBucket(N, torch.float32) if use_nvls else None
    if mcb is not None:
        mcb.tensor.normal_()
    ctx = ta.init_distributed_context(heap_bytes=N * es)
    bucket = ta.bucket_tensor(ctx, N, tdt)
    bucket.normal_()
    for mb in sizes:
        n = max(8, int(mb * 2**20) // es)
        n -= n % 8
        def op():
            if mcb is not None:
                ta.weighted_allreduce_nvls(ctx, mcb, 1.0 / world, view=mcb.tensor[:n])
            else:
                ta.weighted_allreduce(ctx, bucket[:n], 1.0 / world)
        for _ in range(5):
            op()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        op()
        e1.record()
        torch.cuda.synchronize()
        tr = ctx.trace()
        t0 = min(t[0] for t in tr)
        ph = lambda k: [(t[k + 1] - t[k]) / 1e3 for t in tr]  # noqa: E731
        start_spread = (max(t[0] for t in tr) - t0) / 1e3
        last = max(tr, key=lambda t: t[4])
        out = {"rank": rank, "nvls": use_nvls, "dyn": dyn, "bucket_MB": mb, "ctas": len(tr), "event_us": round(e0.elapsed_time(e1) * 1e3, 1),
               "start_spread_us": round(start_spread, 2),
               "entry_med": round(statistics.median(ph(0)), 2), "entry_max": round(max(ph(0)), 2),
               "data_med": round(statistics.median(ph(1)), 2), "data_max": round(max(ph(1)), 2),
               "exit_med": round(statistics.median(ph(2)), 2), "exit_max": round(max(ph(2)), 2),
               "final_us": round((last[4] - last[3]) / 1e3, 2),
               "span_us": round((last[4] - t0) / 1e3, 2)}
        objs = [None] * world
        dist.all_gather_object(objs, out)
        if rank == 0:
            for o in objs:
                print(json.dumps(o), flush=True)
        ctx.gns_stats()
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
