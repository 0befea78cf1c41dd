#!/usr/bin/env python
"""Is K2's tail a per-SM property?  Runs the C4 K2 launch R times, records per CTA its SM
(%smid) and data-done time, and reports per SM the latest done time per launch, how stable the
SM ranking is across launches (Spearman correlation), and the spread.  python tools/k2_smtrace.py"""
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cannikin_synth as synth  # noqa: E402
import paper_2402_05302_b200 as ck  # noqa: E402
from paper_2402_05302_b200 import torch_api as ta  # noqa: E402


def main():
    torch.cuda.set_device(0)
    nr, N, dt = 8, 110_000_000, "bf16"
    b = list(range(1, nr + 1))
    r = [x / sum(b) for x in b]
    gs = synth.device_gns_gradients(nr, N, b, seed=1, dtype=dt)
    out = torch.empty_like(gs[0])
    st = torch.zeros(nr + 1, dtype=torch.float64, device="cuda")
    ctx = ck.Context(world=1, device=0)
    per_launch = []
    for rep in range(8):
        ta.weighted_sum_local(ctx, gs, r, out, st[:nr], st[nr:], variant="ldg")
        ta.weighted_sum_local(ctx, gs, r, out, st[:nr], st[nr:], variant="ldg")
        torch.cuda.synchronize()
        tr = ctx.trace()
        t0 = min(t[0] for t in tr)
        sm_done = {}
        cta_done = []
        for t in tr:
            sm = int(t[1])
            d = (t[2] - t0) / 1e3
            cta_done.append(d)
            sm_done[sm] = max(sm_done.get(sm, 0.0), d)
        per_launch.append(sm_done)
        print(json.dumps({"launch": rep, "ctas": len(tr), "sms": len(sm_done),
                          "sm_done_min": round(min(sm_done.values()), 1),
                          "sm_done_med": round(statistics.median(sm_done.values()), 1),
                          "sm_done_max": round(max(sm_done.values()), 1),
                          "slowest_sms": sorted(sm_done, key=sm_done.get)[-6:]}), flush=True)
    sms = sorted(set.intersection(*[set(d) for d in per_launch]))
    M = np.array([[d[s] for s in sms] for d in per_launch])
    ranks = np.argsort(np.argsort(M, axis=1), axis=1)
    corr = np.corrcoef(ranks)
    off = corr[~np.eye(len(per_launch), dtype=bool)]
    mean_by_sm = M.mean(axis=0)
    print(json.dumps({"spearman_between_launches_mean": round(float(off.mean()), 3),
                      "per_sm_mean_done_spread_us": round(float(mean_by_sm.max() - mean_by_sm.min()), 1),
                      "within_sm_launch_to_launch_sd_us": round(float(M.std(axis=0).mean()), 2),
                      "consistently_slow_sms": [sms[i] for i in np.argsort(mean_by_sm)[-8:]]}))


if __name__ == "__main__":
    main()
