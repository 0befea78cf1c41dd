"""Per-rank worker for tests/test_gpu_nvls.py: cannikin_weighted_allreduce_nvls on a torch
symmetric-memory (multicast) bucket; saves output bits and statistics per case."""
import argparse
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import cannikin_synth as synth  # noqa: E402
import paper_2402_05302_b200 as ck  # noqa: E402
from paper_2402_05302_b200 import torch_api as ta  # noqa: E402
from mp_allreduce_worker import b_for, from_dev, to_dev  # noqa: E402

CASES = [("v1", 8, "f32", 1), ("small", 4096, "f32", 2), ("mid_f32", 1 << 20, "f32", 3),
         ("big_f32", 3_000_000, "f32", 5), ("resnet18", 11_689_512, "f32", 6)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    lr = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(lr)
    dist.init_process_group("nccl", device_id=torch.device("cuda", lr))
    ctx = ta.init_distributed_context(heap_bytes=1 << 20)
    tdt = {"f32": torch.float32, "bf16": torch.bfloat16}
    mcbs = {dt: ta.McBucket(12_000_000, tdt[dt]) for dt in ("f32", "bf16")}
    try:  # bf16 is refused (the switch's bf16 sum misses the tolerance)
        ta.weighted_allreduce_nvls(ctx, mcbs["bf16"], 0.5, view=mcbs["bf16"].tensor[:64])
        bf16 = "accepted"
    except ck.CannikinError as e:
        bf16 = e.name
    np.save(os.path.join(args.out, f"rank{rank}_bf16.npy"), np.array([bf16]))
    for name, N, dtype, seed in CASES:
        b = b_for(world, seed)
        B = sum(b)
        gs = synth.gns_gradients(world, N, b, seed=seed, dtype=dtype)
        mcb = mcbs[dtype]
        view = mcb.tensor[:N]
        outs, stats = [], []
        for rep in range(2):
            view.copy_(to_dev(gs[rank], dtype))
            ta.weighted_allreduce_nvls(ctx, mcb, b[rank] / B, view=view)
            loc, glob = ctx.gns_stats()
            outs.append(from_dev(view, dtype))
            stats.append((loc, glob))
        np.savez(os.path.join(args.out, f"rank{rank}_{name}.npz"), out1=outs[0], out2=outs[1],
                 loc=np.array(stats[0][0]), glob=stats[0][1], loc2=np.array(stats[1][0]),
                 glob2=stats[1][1], b=np.array(b))
    # ragged sizes are refused, not silently mishandled
    try:
        ta.weighted_allreduce_nvls(ctx, mcbs["f32"], 0.5, view=mcbs["f32"].tensor[:7])
        ragged = "accepted"
    except ck.CannikinError as e:
        ragged = e.name
    np.save(os.path.join(args.out, f"rank{rank}_ragged.npy"), np.array([ragged]))
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
