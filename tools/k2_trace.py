#!/usr/bin/env python
"""Device timeline of the emulated-rank kernel (K2, LDG variant) from its %globaltimer trace:
CTA start spread (launch ramp), distribution of CTA data-done times (tail imbalance), final
reduction.  python tools/k2_trace.py"""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cannikin_synth as synth  # noqa: E402
import paper_2402_05302_b200 as ck  # noqa: E402
from paper_2402_05302_b200 import torch_api as ta  # noqa: E402


def q(xs, p):
    xs = sorted(xs)
    return xs[min(len(xs) - 1, int(p * len(xs)))]


def main():
    torch.cuda.set_device(0)
    nt = os.environ.get("CANNIKIN_K2_NT", "256")
    for name, nr, N, dt in [("c4", 8, 110_000_000, "bf16"), ("c5", 8, 354_823_168, "f32"),
                            ("c4q", 8, 27_500_000, "bf16")]:
        b = list(range(1, nr + 1))
        r = [x / sum(b) for x in b]
        gs = synth.device_gns_gradients(nr, N, b, seed=1, dtype=dt)
        out = torch.empty_like(gs[0])
        st = torch.zeros(nr + 1, dtype=torch.float64, device="cuda")
        ctx = ck.Context(world=1, device=0)
        for _ in range(5):
            ta.weighted_sum_local(ctx, gs, r, out, st[:nr], st[nr:], variant="ldg")
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ta.weighted_sum_local(ctx, gs, r, out, st[:nr], st[nr:], variant="ldg")  # queue ahead
        e0.record()
        ta.weighted_sum_local(ctx, gs, r, out, st[:nr], st[nr:], variant="ldg")
        e1.record()
        torch.cuda.synchronize()
        tr = ctx.trace()
        t0 = min(t[0] for t in tr)
        starts = [(t[0] - t0) / 1e3 for t in tr]
        done = [(t[2] - t0) / 1e3 for t in tr]
        last = max(tr, key=lambda t: t[4])
        nbytes = (nr + 1) * N * (4 if dt == "f32" else 2)
        print(json.dumps({"shape": name, "nt": nt, "ctas": len(tr), "event_us": round(e0.elapsed_time(e1) * 1e3, 1),
                          "start_spread_us": round(max(starts), 2),
                          "done_min": round(min(done), 1), "done_med": round(statistics.median(done), 1),
                          "done_p90": round(q(done, 0.9), 1), "done_max": round(max(done), 1),
                          "end_us": round((last[4] - t0) / 1e3, 1),
                          "last_cta_blocksum_us": round((last[3] - last[2]) / 1e3, 2),
                          "last_cta_final_us": round((last[4] - last[3]) / 1e3, 2),
                          "GBps_at_median_done": round(nbytes / (statistics.median(done) * 1e-6) / 1e9),
                          "GBps_span": round(nbytes / ((last[4] - t0) * 1e-9) / 1e9)}), flush=True)
        ctx.close()
        del gs, out


if __name__ == "__main__":
    main()
