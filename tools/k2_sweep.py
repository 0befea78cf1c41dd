#!/usr/bin/env python
"""Kernel-time sweep of the emulated-rank pass (K2) variants on one GPU.

Each configuration is captured as a CUDA graph of R back-to-back launches bracketed by timing
events (no host gaps); reports median per-launch time and algorithmic GB/s = (n+1) N s / t.
    python tools/k2_sweep.py [--reps 10]
"""
import argparse
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cannikin_synth as synth  # noqa: E402
import paper_2402_05302_b200 as ck  # noqa: E402
from paper_2402_05302_b200 import torch_api as ta  # noqa: E402

SHAPES = [("c1", 3, 1 << 20, "f32"), ("c4", 8, 110_000_000, "bf16"), ("c5", 8, 354_823_168, "f32"), ("c3", 8, 25_557_032, "f32"),
          ("c2", 2, 11_689_512, "f32"), ("c1-big", 3, 1 << 26, "f32"), ("c4x3", 3, 110_000_000, "bf16"),
          ("c4f32", 8, 110_000_000, "f32"), ("c5bf16", 8, 354_823_168, "bf16"),
          ("c4x2", 8, 220_000_000, "bf16"), ("c4q", 8, 27_500_000, "bf16"),
          ("c4h", 8, 55_000_000, "bf16")]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--shapes", default="c4,c5,c3,c2,c1-big,c4x3")
    ap.add_argument("--grids", default="0,148,296,444,592,740,888")
    ap.add_argument("--altu-grids", default="0")
    ap.add_argument("--tma", type=int, default=1)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    want = args.shapes.split(",")
    for name, nr, N, dt in SHAPES:
        if name not in want:
            continue
        b = list(range(1, nr + 1))
        r = [x / sum(b) for x in b]
        gs = synth.device_gns_gradients(nr, N, b, seed=1, dtype=dt)
        out = torch.empty_like(gs[0])
        st = torch.zeros(nr + 1, dtype=torch.float64, device="cuda")
        nbytes = (nr + 1) * N * (4 if dt == "f32" else 2)
        variants = [("tma", None, 0)] if args.tma else []
        variants += [("ldg", int(g), 0) for g in args.grids.split(",")]
        variants += [("ldg", int(g), 1) for g in args.altu_grids.split(",") if g]
        for var, grid, altu in variants:
            if grid is not None:
                os.environ["CANNIKIN_LOCAL_GRID"] = str(grid)
            os.environ["CANNIKIN_K2_NT"] = "1024" if altu else "256"
            ctx = ck.Context(world=1, device=0)
            for _ in range(3):
                ta.weighted_sum_local(ctx, gs, r, out, st[:nr], st[nr:], variant=var)
            torch.cuda.synchronize()
            evs = [(torch.cuda.Event(enable_timing=True, external=True),
                    torch.cuda.Event(enable_timing=True, external=True)) for _ in range(args.reps)]
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for e0, e1 in evs:
                    e0.record()
                    ta.weighted_sum_local(ctx, gs, r, out, st[:nr], st[nr:], variant=var)
                    e1.record()
            times = []
            for _ in range(3):
                g.replay()
                torch.cuda.synchronize()
                times += [a.elapsed_time(c) for a, c in evs]
            t = statistics.median(times)
            print(json.dumps({"shape": name, "ranks": nr, "N": N, "dtype": dt, "variant": var,
                              "grid": grid, "nt1024": altu,
                              "ms": round(t, 4),
                              "GBps": round(nbytes / (t * 1e-3) / 1e9, 1)}), flush=True)
            del g
            ctx.close()
        del gs, out


if __name__ == "__main__":
    main()
