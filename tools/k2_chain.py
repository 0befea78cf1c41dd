#!/usr/bin/env python
"""K2 in the bucketed regime: the C4 gradient (8 emulated ranks, 110M bf16) cut into buckets of
--bucket-mb, one cannikin_weighted_sum_local per bucket, with and without PDL chaining
(CANNIKIN_LOCAL_CHAIN), in a CUDA graph and eagerly.  Prints one JSON line per configuration:
chain time (first start to last end, CUDA events), GB/s on K2's (n+1) N s bytes, fraction of the
measured HBM peak."""
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bucket-mb", default="0,100,50,25,10")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--config", default="c4")
    ap.add_argument("--gaps-ms", default="", help="whole-gradient launches with idle gaps between "
                    "them (e.g. 0,1,10,100): does the per-launch time depend on the duty cycle?")
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    N, n, dt = cfg["N"], cfg["n_emu"], cfg["dtype"]
    s = bench.esize(dt)
    tdt = {"f32": torch.float32, "bf16": torch.bfloat16}[dt]
    b = ck.opt_split(bench.node_models(n), bench.COMM, cfg["B"])["b"]
    r = [x / sum(b) for x in b]
    ctx = ck.Context(world=1, device=0)
    gs = synth.device_gns_gradients(n, N, b, seed=0, dtype=dt)
    out = torch.empty(N, dtype=tdt, device="cuda")
    st = torch.zeros(n + 1, dtype=torch.float64, device="cuda")
    peak = bench.measured_peaks()[0]["hbm_gbs"]
    if args.gaps_ms:
        import time

        def one():
            ta.weighted_sum_local(ctx, gs, r, out, st[:n], st[n:])
        for _ in range(5):
            one()
        torch.cuda.synchronize()
        for gap in [float(x) for x in args.gaps_ms.split(",")]:
            ts = []
            for it in range(args.reps + 50):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                one()
                e1.record()
                if gap > 0:
                    torch.cuda.synchronize()
                    time.sleep(gap * 1e-3)
                ts.append((e0, e1))
            torch.cuda.synchronize()
            v = sorted(a.elapsed_time(c) for a, c in ts[50:])
            print(json.dumps({"gap_ms": gap, "kernel_ms_p50": round(v[len(v) // 2], 4),
                              "kernel_ms_min": round(v[0], 4), "kernel_ms_max": round(v[-1], 4),
                              "GBs_p50": round((n + 1) * N * s / (v[len(v) // 2] * 1e-3) / 1e9, 1)}),
                  flush=True)
        return
    for mb in [float(x) for x in args.bucket_mb.split(",")]:
        be = N if mb <= 0 else int(mb * 2**20) // s
        be -= be % 8
        cuts = list(range(0, N, be)) + [N]
        nb = len(cuts) - 1
        for chain in (False, True):
            def seq():
                for i in range(nb):
                    a, c = cuts[i], cuts[i + 1]
                    ta.weighted_sum_local(ctx, [g[a:c] for g in gs], r, out[a:c], st[:n], st[n:],
                                          accumulate=i > 0, chain=chain and i > 0)
            for mode in ("graph", "eager"):
                seq()
                torch.cuda.synchronize()
                if mode == "graph":
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g):
                        seq()
                    run = g.replay
                else:
                    run = seq
                for _ in range(3):
                    run()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                ts = []
                for _ in range(args.reps):
                    e0.record()
                    run()
                    e1.record()
                    torch.cuda.synchronize()
                    ts.append(e0.elapsed_time(e1))
                ts.sort()
                med = ts[len(ts) // 2]
                gbs = (n + 1) * N * s / (med * 1e-3) / 1e9
                print(json.dumps({"bucket_mb": mb, "launches": nb, "chain": chain, "mode": mode,
                                  "ms": round(med, 4), "ms_min": round(ts[0], 4),
                                  "per_launch_us": round(med * 1e3 / nb, 2),
                                  "GBs": round(gbs, 1), "frac": round(gbs / peak, 4)}), flush=True)


if __name__ == "__main__":
    main()
