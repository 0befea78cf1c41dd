#!/usr/bin/env python
"""Characterise the NVSwitch bf16 reduction (why the NVLS path K6 is fp32-only; Q28).

    torchrun --nproc-per-node W tools/nvls_bf16_probe.py [--n 4000000]

Runs cannikin_weighted_allreduce_nvls on a bf16 bucket (CANNIKIN_NVLS_BF16=1 lets the library
accept it) and compares, on rank 0:
  * the Q1 error of the result against the oracle's Eq. 9 (the bf16 tolerance is 1e-2);
  * the switch's sum against RN_bf16(exact sum of the phase-A inputs y_j = RN_bf16(r_j g_j)), the
    result an fp32-accumulating switch with one round-to-nearest-even would return: fraction of
    identical bits, ulp histogram and sign of the differences (truncation shows up as one sign).
Prints one JSON line."""
import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["CANNIKIN_NVLS_BF16"] = "1"
os.environ.setdefault("CANNIKIN_SPIN_TIMEOUT_MS", "60000")
import cannikin_synth as synth  # noqa: E402
from oracle import aggregate as agg  # noqa: E402
from paper_2402_05302_b200 import torch_api as ta  # noqa: E402


def bits(t):
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4_000_000)
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    lr = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(lr)
    dist.init_process_group("nccl", device_id=torch.device("cuda", lr))
    ctx = ta.init_distributed_context(heap_bytes=1 << 20)
    N = args.n - args.n % 8
    b = [int(x) for x in np.random.default_rng(5).integers(1, 97, size=world)]
    r = agg.ratios(b)
    gs = synth.device_gns_gradients(world, N, b, seed=3, dtype="bf16")
    mcb = ta.McBucket(N, torch.bfloat16)
    mcb.tensor.copy_(gs[rank])
    torch.cuda.synchronize()
    dist.barrier()
    ta.weighted_allreduce_nvls(ctx, mcb, float(r[rank]))
    ctx.gns_stats()
    out = mcb.tensor.clone()
    if rank == 0:
        ins = [agg.to_f64(bits(g), "bf16") for g in gs]
        ref = agg.weighted_sum(ins, r)
        scale = np.maximum(agg.elementwise_scale(ins, r), 1e-30)
        got = agg.to_f64(bits(out), "bf16")
        q1 = float(np.max(np.abs(got - ref) / scale))
        # phase A as the kernel computes it: fp32 product, one RN to bf16
        ys = [(torch.tensor(float(np.float32(r[j])), device="cuda") * gs[j].float()).to(torch.bfloat16)
              for j in range(world)]
        exact = sum(agg.to_f64(bits(y), "bf16") for y in ys)  # W bf16 values: exact in float64
        rn = torch.from_numpy(exact).cuda().float().to(torch.bfloat16)  # f64->f32 exact here? see note
        want, have = bits(rn).astype(np.int32), bits(out).astype(np.int32)
        # ulp distance on the sign-magnitude bf16 encoding
        def ordered(u):
            return np.where(u & 0x8000, -(u & 0x7FFF), u & 0x7FFF)
        d = ordered(have) - ordered(want)
        nz = d[d != 0]
        res = {"world": world, "N": N, "b": b, "q1_err": q1, "tolerance": 1e-2,
               "identical_to_rn_of_exact_sum": float(np.mean(d == 0)),
               "ulp_hist": {int(k): int(v) for k, v in zip(*np.unique(np.clip(d, -4, 4),
                                                                        return_counts=True))},
               "diff_sign": {"pos": int(np.sum(nz > 0)), "neg": int(np.sum(nz < 0))},
               "toward_zero": int(np.sum((np.abs(agg.to_f64(have.astype(np.uint16), "bf16"))
                                          < np.abs(agg.to_f64(want.astype(np.uint16), "bf16"))))),
               "note": "RN of the exact phase-A sum computed as f64 -> f32 -> bf16 (double "
                       "rounding possible only where the f64 sum is not an f32)"}
        print(json.dumps(res), flush=True)
    dist.barrier()
    del mcb
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
