#!/usr/bin/env python
"""BASELINE configs[3] loop: BERT-base-sized gradient (110M bf16) with the total batch adapted by
the heterogeneous GNS (§4.4; goodput P:143; OptPerf_init P:410-415).

    python tools/adaptive_batch.py                      (1 GPU: 8 emulated ranks, K2)
    torchrun --nproc-per-node N tools/adaptive_batch.py (N GPUs, K3)

Synthetic training: the true noise scale trS/|G|^2 follows a rising schedule (50 -> 5000 over the
epochs, the "batch size grows as training converges" shape of fig:gns).  Every step each rank draws
its mean gradient for its b_i from the V1 recipe (cannikin_synth), the hot path reduces it and
returns the norm statistics, the host estimates G and S (Theorem 1) and updates the EMA.  At the
end of each epoch the analyzer picks the next total batch by goodput over the candidate list and
splits it with opt_split (node models of bench.py's emulated mix, comm model of the measured
kernels).  Rank 0 prints one JSON line per epoch.
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import cannikin_synth as synth  # noqa: E402
import paper_2402_05302_b200 as ck  # noqa: E402
from paper_2402_05302_b200 import torch_api as ta  # noqa: E402

CANDS = [9, 16, 32, 64, 96, 128, 192, 256, 384, 512, 768, 1024]


def main():
    os.environ.setdefault("CANNIKIN_SPIN_TIMEOUT_MS", "120000")  # report, do not hang
    ap = argparse.ArgumentParser()
    ap.add_argument("--epochs", type=int, default=8)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--N", type=int, default=110_000_000)
    ap.add_argument("--emulated", type=int, default=8)
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    lr = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(lr)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", lr))
    n = world if world > 1 else args.emulated
    N = args.N
    models = bench.hetero_models(n)
    comm = (1.0 / 9, 8 * 65e-6, 65e-6)  # gamma = 1/buckets, T_o, T_u of ~25 MB K3 buckets
    B0 = CANDS[0]
    B = max(B0, n)
    if world > 1:
        ctx = ta.init_distributed_context(heap_bytes=N * 2)
        bucket = ta.bucket_tensor(ctx, N, torch.bfloat16)
    else:
        ctx = ck.Context(world=1, device=0)
        out = torch.empty(N, dtype=torch.bfloat16, device="cuda")
        stats = torch.zeros(n + 1, dtype=torch.float64, device="cuda")
    ema = ck.GnsEma(0.9)
    sched = [50.0 * (100.0 ** (e / max(1, args.epochs - 1))) for e in range(args.epochs)]
    for epoch in range(args.epochs):
        trS = sched[epoch]
        split = ck.opt_split(models, comm, B)["b"]
        est_last = None
        for step in range(args.steps):
            seed = 1000 * epoch + step
            if world > 1:
                g = synth.device_gns_gradients(n, N, split, G2=1.0, trS=trS, seed=seed,
                                               dtype="bf16", ranks=[rank])[0]
                bucket.copy_(g)
                del g
                ta.weighted_allreduce(ctx, bucket, split[rank] / B)
                loc, gsq = ctx.gns_stats()
            else:
                gs = synth.device_gns_gradients(n, N, split, G2=1.0, trS=trS, seed=seed,
                                                dtype="bf16")
                ta.weighted_sum_local(ctx, gs, [x / B for x in split], out, stats[:n], stats[n:])
                st = stats.tolist()
                loc, gsq = st[:n], st[n]
                del gs
            est = ck.gns_estimate(loc, gsq, split)
            ema.update(est["G2"], est["trS"])
            est_last = est
        Bn = ema.B_noise
        nxt = ck.choose_batch(models, comm, CANDS, B0, Bn)
        if rank == 0:
            print(json.dumps({"epoch": epoch, "B": B, "split": split, "true_B_noise": round(trS, 2),
                              "est_B_noise_last_step": round(est_last["B_noise"], 2),
                              "ema_B_noise": round(Bn, 2), "next_B": nxt["B"],
                              "goodput_next": round(max(nxt["goodput"]), 2),
                              "ranks": n, "emulated": world == 1}), flush=True)
        B = nxt["B"]
    if dist is not None:
        dist.barrier()
        ctx.close()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
