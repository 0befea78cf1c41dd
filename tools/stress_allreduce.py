#!/usr/bin/env python
"""Stress of the flag protocols (two-shot barriers, LL's 8-byte words, LL128's 128-byte lines):
many back-to-back weighted all-reduces of seeded random sizes, every result checked bit for bit.

Inputs are chosen so that Eq. 9 is EXACT in fp32 and bf16: rank j's bucket holds small integers
(j + 1) * ((e * 7 + call) mod 13 - 6) and the shares are dyadic (b_j = 2^k_j, B a power of two),
so sum_j r_j g_j[e] has an exact bf16 / fp32 value computed here in torch on the device; any lost,
torn or stale line shows up as a mismatch.  No host sync between calls inside a batch (the
epochs and parities of consecutive calls overlap as in a training step); a batch is checked
after it completes.
    torchrun --nproc-per-node N tools/stress_allreduce.py [--calls 20000] [--variant auto|ll|ll128|twoshot]
Rank 0 prints one JSON line: calls, elements moved, mismatching calls (must be 0)."""
import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_05302_b200 as ck  # noqa: E402
from paper_2402_05302_b200 import torch_api as ta  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--calls", type=int, default=20000)
    ap.add_argument("--batch", type=int, default=20)
    ap.add_argument("--variant", default="auto", choices=["auto", "ll", "ll128", "twoshot"])
    ap.add_argument("--max-elems", type=int, default=4 << 20)
    ap.add_argument("--gated", action="store_true", help="CANNIKIN_INIT_GATED_ENTRY, a late rank")
    args = ap.parse_args()
    knobs = {"ll": ("1", "0"), "ll128": ("0", "1"), "twoshot": ("0", "0")}
    if args.variant in knobs:
        os.environ["CANNIKIN_AR_LL"], os.environ["CANNIKIN_AR_LL128"] = knobs[args.variant]
    os.environ.setdefault("CANNIKIN_SPIN_TIMEOUT_MS", "60000")
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    lr = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(lr)
    dist.init_process_group("nccl", device_id=torch.device("cuda", lr))
    ctx = ta.init_distributed_context(heap_bytes=args.max_elems * 4 * args.batch + (1 << 20),
                                      gated=args.gated)
    rng = np.random.default_rng(1234)  # same sequence on every rank
    bad, done, moved = 0, 0, 0
    while done < args.calls:
        jobs = []
        for _ in range(args.batch):
            n = int(rng.integers(1, args.max_elems // 8)) * 8
            dt = torch.bfloat16 if rng.random() < 0.5 else torch.float32
            k = rng.integers(0, 4, size=world)
            b = [1 << int(x) for x in k]
            B = sum(b)
            pw = 1 << int(np.ceil(np.log2(B)))
            r = [x / pw for x in b]  # dyadic shares (sum <= 1 is fine: no ratio check here)
            jobs.append((n, dt, r))
        bufs = []
        for t, (n, dt, r) in enumerate(jobs):
            e = torch.arange(n, device="cuda", dtype=torch.int64)
            pat = ((e * 7 + done + t) % 13 - 6).to(torch.float32)
            x = ta.bucket_tensor(ctx, n, dt)
            x.copy_((pat * (rank + 1)).to(dt))
            want = (pat * sum(r[j] * (j + 1) for j in range(world))).to(dt)
            bufs.append((x, want))
        torch.cuda.synchronize()
        dist.barrier()
        for t, ((x, _), (n, dt, r)) in enumerate(zip(bufs, jobs)):
            if args.gated and rank == (done + t) % world and t % 5 == 0:
                ck.emulate_compute(2e-4, torch.cuda.current_stream().cuda_stream)  # late rank
            ta.weighted_allreduce(ctx, x, r[rank])
        torch.cuda.synchronize()
        ctx.gns_stats()
        for x, want in bufs:
            if not torch.equal(x.view(torch.int16) if x.dtype == torch.bfloat16 else x,
                               want.view(torch.int16) if want.dtype == torch.bfloat16 else want):
                bad += 1
            moved += x.numel()
            ta.free_bucket_tensor(ctx, x)
        done += len(jobs)
    t = torch.tensor([bad, done, moved], device="cuda", dtype=torch.float64)
    dist.all_reduce(t)
    if rank == 0:
        print(json.dumps({"world": world, "variant": args.variant, "gated": args.gated,
                          "calls": int(t[1].item()) // world,
                          "elements": int(t[2].item()) // world, "mismatching_calls": int(t[0].item()),
                          "max_elems": args.max_elems}), flush=True)
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
