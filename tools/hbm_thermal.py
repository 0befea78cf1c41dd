#!/usr/bin/env python
"""Is the 8-9% swing of the 8:1 memory pattern (and of K2) on one box a thermal / memory-state
effect?  tools/k2_placement.py saw the same buffers run 0.286 or 0.313 ms depending on which case
came before.  Here the bare pattern (tools/pattern_kernel.cu, C4 shape) and K2 are timed
repeatedly on ONE set of buffers with fixed contents while the HBM is heated (K2 back to back for
a few seconds) and left to cool (idle), with nvidia-smi's GPU / memory temperature, memory clock
and power sampled at every point.  One JSON line per point.
    python tools/hbm_thermal.py"""
import ctypes
import json
import os
import subprocess
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import cannikin_synth as synth  # noqa: E402
import paper_2402_05302_b200 as ck  # noqa: E402
from paper_2402_05302_b200 import torch_api as ta  # noqa: E402
from k2_vs_pattern import pattern_lib, timed  # noqa: E402

n, N = 8, 110_000_000


def smi():
    q = ("temperature.gpu,temperature.memory,clocks.mem,clocks.sm,power.draw,"
         "clocks_event_reasons.active")
    out = subprocess.run(["nvidia-smi", "-i", "0", f"--query-gpu={q}", "--format=csv,noheader,nounits"],
                         capture_output=True, text=True).stdout.strip().split(", ")
    return dict(zip(q.split(","), out))


def main():
    torch.cuda.set_device(0)
    bufs = [torch.empty(N, dtype=torch.bfloat16, device="cuda").normal_() for _ in range(n + 1)]
    gs, out = bufs[:n], bufs[n]
    P = pattern_lib()
    ptrs = (ctypes.c_void_p * n)(*[g.data_ptr() for g in gs])
    ctx = ck.Context(world=1, device=0)
    st = torch.zeros(n + 1, dtype=torch.float64, device="cuda")
    b = list(range(1, n + 1))
    r = [x / sum(b) for x in b]
    nbytes = (n + 1) * N * 2

    def pat():
        P.pattern_launch(ptrs, n, out.data_ptr(), N * 2, 592,
                         ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))

    def k2():
        ta.weighted_sum_local(ctx, gs, r, out, st[:n], st[n:])

    t_start = time.time()

    # the driver's roofline denominator, in the same state: torch copy of 1 Gi bf16 elements
    ca = torch.empty(1 << 30, dtype=torch.bfloat16, device="cuda").normal_()
    cb = torch.empty_like(ca)

    def point(tag):
        ms_p = timed(pat)
        ms_k = timed(k2)
        ms_c = timed(lambda: cb.copy_(ca), reps=10, rounds=2)
        print(json.dumps({"t_s": round(time.time() - t_start, 2), "phase": tag,
                          "pattern_ms": round(ms_p, 4), "k2_ms": round(ms_k, 4),
                          "k2_GBs": round(nbytes / ms_k / 1e6, 1),
                          "copy_GBs": round(4 * (1 << 30) / ms_c / 1e6, 1), **smi()}), flush=True)

    def heat(seconds):
        t0 = time.time()
        while time.time() - t0 < seconds:
            for _ in range(200):
                k2()
            torch.cuda.synchronize()

    for data in ("normal", "synth"):
        if data == "synth":
            for g, x in zip(gs, synth.device_gns_gradients(n, N, b, seed=1, dtype="bf16")):
                g.copy_(x)
            torch.cuda.empty_cache()
        for i in range(3):
            point(f"{data}: start {i}")
        for i in range(4):
            heat(3.0)
            point(f"{data}: after {3 * (i + 1)} s of K2")
        for i in range(4):
            time.sleep(5.0)
            point(f"{data}: idle {5 * (i + 1)} s")
        if data == "normal":
            time.sleep(40.0)
            point("normal: idle 60 s")

    def heat_smi(seconds):  # the throttle reasons while the heat runs
        t0 = time.time()
        rs = []
        while time.time() - t0 < seconds:
            for _ in range(100):
                k2()
            rs.append(smi())
            torch.cuda.synchronize()
        return rs
    print(json.dumps({"during_k2": heat_smi(2.0)}), flush=True)


if __name__ == "__main__":
    main()
