#!/usr/bin/env python
"""K2 against the bare memory pattern it is bound by, on the SAME buffers in the same run.

tools/hbm_probe*.cu measured the 8-read + 1-write 16-byte stream (no arithmetic) at 6.2-7.0 TB/s
depending on the box and on where the 9 streams sit in physical memory; box-to-box spread makes
cross-run comparisons useless.  Here K2 (cannikin_weighted_sum_local, C4: 8 x 110M bf16) and the
pattern kernel (tools/pattern_kernel.cu, integer adds) are timed back to back on the bench's own
inputs (cannikin_synth tensors) and on freshly allocated ones, at several grids.  One JSON line per
case: median per-launch ms over graphs of R back-to-back launches, GB/s on (n+1) N s bytes.
    python tools/k2_vs_pattern.py"""
import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import cannikin_synth as synth  # noqa: E402
import paper_2402_05302_b200 as ck  # noqa: E402
from paper_2402_05302_b200 import torch_api as ta  # noqa: E402


def pattern_lib():
    so = "/tmp/cannikin_pattern.so"
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared",
                           "-Xcompiler", "-fPIC", "-o", so,
                           os.path.join(ROOT, "tools", "pattern_kernel.cu")])
    L = ctypes.CDLL(so)
    L.pattern_launch.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int, ctypes.c_void_p,
                                 ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
    return L


def timed(fn, reps=20, rounds=3):
    fn()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True, external=True),
            torch.cuda.Event(enable_timing=True, external=True)) for _ in range(reps)]
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for e0, e1 in evs:
            e0.record()
            fn()
            e1.record()
    ts = []
    for _ in range(rounds):
        g.replay()
        torch.cuda.synchronize()
        ts += [a.elapsed_time(b) for a, b in evs]
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sets", default="synth,fresh,one_alloc")
    ap.add_argument("--k2-grids", default="0,444,592,740,888")
    ap.add_argument("--pattern-grids", default="444,592,740,888")
    ap.add_argument("--tag", default=os.environ.get("CANNIKIN_LIB", "in-tree"))
    args = ap.parse_args()
    sets = args.sets.split(",")
    torch.cuda.set_device(0)
    n, N = 8, 110_000_000
    nbytes = (n + 1) * N * 2
    P = pattern_lib()
    b = list(range(1, n + 1))
    r = [x / sum(b) for x in b]

    def run_set(tag, gs, out):
        st = torch.zeros(n + 1, dtype=torch.float64, device="cuda")
        ptrs = (ctypes.c_void_p * n)(*[g.data_ptr() for g in gs])
        for grid in [int(g) for g in args.k2_grids.split(",") if g]:
            os.environ["CANNIKIN_LOCAL_GRID"] = str(grid)
            for nt in ("256", "1024") if grid == 0 else ("256",):
                os.environ["CANNIKIN_K2_NT"] = nt
                ctx = ck.Context(world=1, device=0)
                ms = timed(lambda: ta.weighted_sum_local(ctx, gs, r, out, st[:n], st[n:]))
                torch.cuda.synchronize()
                ctas = len(ctx.trace())
                print(json.dumps({"lib": args.tag, "buffers": tag, "kernel": "k2", "grid": grid,
                                  "ctas": ctas, "nt": int(nt),
                                  "ms": round(ms, 4), "GBs": round(nbytes / ms / 1e6, 1)}), flush=True)
                ctx.close()
        os.environ["CANNIKIN_LOCAL_GRID"] = "0"
        os.environ["CANNIKIN_K2_NT"] = "256"
        for grid in [int(g) for g in args.pattern_grids.split(",") if g]:
            def pat():
                rc = P.pattern_launch(ptrs, n, out.data_ptr(), N * 2, grid,
                                      ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
                assert rc == 0, rc
            ms = timed(pat)
            print(json.dumps({"lib": args.tag, "buffers": tag, "kernel": "pattern", "grid": grid,
                              "ms": round(ms, 4), "GBs": round(nbytes / ms / 1e6, 1)}), flush=True)

    if "synth" in sets:
        gs = synth.device_gns_gradients(n, N, b, seed=1, dtype="bf16")
        out = torch.empty_like(gs[0])
        run_set("synth", gs, out)
        del gs, out
        torch.cuda.empty_cache()
    if "fresh" in sets:
        gs = [torch.empty(N, dtype=torch.bfloat16, device="cuda").normal_() for _ in range(n)]
        out = torch.empty(N, dtype=torch.bfloat16, device="cuda")
        run_set("fresh", gs, out)
        del gs, out
        torch.cuda.empty_cache()
    if "one_alloc" not in sets:
        return
    # one allocation, streams 2 MiB-rounded apart
    per = (N * 2 + (2 << 20) - 1) // (2 << 20) * (2 << 20) // 2
    big = torch.empty(per * (n + 1), dtype=torch.bfloat16, device="cuda").normal_()
    gs = [big[j * per: j * per + N] for j in range(n)]
    out = big[n * per: n * per + N]
    run_set("one_alloc", gs, out)


if __name__ == "__main__":
    main()
