#!/usr/bin/env python
"""Small single-GPU cases for compute-sanitizer: K2 (both variants, ragged sizes), world-1
weighted_allreduce, stats readback."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cannikin_synth as synth  # noqa: E402
import paper_2402_05302_b200 as ck  # noqa: E402
from paper_2402_05302_b200 import torch_api as ta  # noqa: E402


def main():
    torch.cuda.set_device(0)
    ctx = ck.Context(world=1, device=0)
    for dt, tdt in (("f32", torch.float32), ("bf16", torch.bfloat16)):
        for nr in (1, 3, 8):
            for N in (0, 1, 7, 4099, 65536 + 5):
                gs = synth.gns_gradients(nr, N, [1] * nr, seed=N, dtype=dt)
                ins = [torch.from_numpy(g.view(np.int16).copy() if dt == "bf16" else g.copy()).cuda()
                       for g in gs]
                if dt == "bf16":
                    ins = [x.view(torch.bfloat16) for x in ins]
                out = torch.empty(N, dtype=tdt, device="cuda")
                st = torch.zeros(nr + 1, dtype=torch.float64, device="cuda")
                for var in ("ldg", "tma"):
                    ta.weighted_sum_local(ctx, ins, [1.0 / nr] * nr, out, st[:nr], st[nr:],
                                          variant=var)
                if N:
                    ta.weighted_allreduce(ctx, ins[0], 1.0)
                torch.cuda.synchronize()
    print(ctx.gns_stats())
    ctx.close()
    print("sanitize cases done")


if __name__ == "__main__":
    main()
