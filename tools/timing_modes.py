#!/usr/bin/env python
"""How much do the timing events themselves cost?  Times the K2 launch of one shape four ways:
graph with an event pair per launch, graph with one pair around R launches, eager with one pair
around R launches, eager with a pair per launch (GPU kept busy)."""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cannikin_synth as synth  # noqa: E402
import paper_2402_05302_b200 as ck  # noqa: E402
from paper_2402_05302_b200 import torch_api as ta  # noqa: E402


def main():
    torch.cuda.set_device(0)
    R = 20
    for name, nr, N, dt, var in [("c4", 8, 110_000_000, "bf16", "ldg"), ("c4", 8, 110_000_000, "bf16", "tma"),
                                 ("c1", 3, 1 << 20, "f32", "ldg"), ("c5", 8, 354_823_168, "f32", "ldg")]:
        b = list(range(1, nr + 1))
        r = [x / sum(b) for x in b]
        gs = synth.device_gns_gradients(nr, N, b, seed=1, dtype=dt)
        out = torch.empty_like(gs[0])
        st = torch.zeros(nr + 1, dtype=torch.float64, device="cuda")
        nbytes = (nr + 1) * N * (4 if dt == "f32" else 2)
        ctx = ck.Context(world=1, device=0)

        def k():
            ta.weighted_sum_local(ctx, gs, r, out, st[:nr], st[nr:], variant=var)

        for _ in range(3):
            k()
        torch.cuda.synchronize()
        res = {}
        # (a) graph, event pair per launch
        evs = [(torch.cuda.Event(enable_timing=True, external=True),
                torch.cuda.Event(enable_timing=True, external=True)) for _ in range(R)]
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for e0, e1 in evs:
                e0.record()
                k()
                e1.record()
        g.replay(); torch.cuda.synchronize()
        g.replay(); torch.cuda.synchronize()
        res["graph_pair_per_launch"] = statistics.median(a.elapsed_time(c) for a, c in evs)
        # (b) graph, one pair around R launches
        e0 = torch.cuda.Event(enable_timing=True, external=True)
        e1 = torch.cuda.Event(enable_timing=True, external=True)
        g2 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g2):
            e0.record()
            for _ in range(R):
                k()
            e1.record()
        g2.replay(); torch.cuda.synchronize()
        g2.replay(); torch.cuda.synchronize()
        res["graph_one_pair"] = e0.elapsed_time(e1) / R
        # (c) eager, one pair around R launches
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        a0.record()
        for _ in range(R):
            k()
        a1.record()
        torch.cuda.synchronize()
        res["eager_one_pair"] = a0.elapsed_time(a1) / R
        # (d) eager, pair per launch, no syncs in between
        pe = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(R)]
        for p0, p1 in pe:
            p0.record()
            k()
            p1.record()
        torch.cuda.synchronize()
        res["eager_pair_per_launch"] = statistics.median(p0.elapsed_time(p1) for p0, p1 in pe)
        # (e) spaced: 2 ms of idle HBM (one spinning warp) before every launch
        pe = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(R)]
        for p0, p1 in pe:
            ck.emulate_compute(2e-3)
            p0.record()
            k()
            p1.record()
        torch.cuda.synchronize()
        res["spaced_2ms"] = statistics.median(p0.elapsed_time(p1) for p0, p1 in pe)
        # (f) L2 flushed (write 256 MB) before every launch, graph-free
        flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
        pe = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(R)]
        for p0, p1 in pe:
            flush.zero_()
            p0.record()
            k()
            p1.record()
        torch.cuda.synchronize()
        res["after_l2_flush"] = statistics.median(p0.elapsed_time(p1) for p0, p1 in pe)
        del flush
        print(json.dumps({"shape": name, "variant": var, "bytes": nbytes,
                          **{m: round(v * 1e3, 2) for m, v in res.items()},
                          **{m + "_GBps": round(nbytes / (v * 1e-3) / 1e9) for m, v in res.items()}}), flush=True)
        ctx.close()
        del gs, out


if __name__ == "__main__":
    main()
