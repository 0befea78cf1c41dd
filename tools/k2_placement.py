#!/usr/bin/env python
"""Where the 9 streams of K2 (C4: 8 x 110M bf16 + output) sit in memory, and what that does to the
kernel, in ONE process (cross-run spread hides it otherwise).  Every case times K2 at its default
grid and the bare 8:1 memory pattern (tools/pattern_kernel.cu) on the same buffers.

  virgin      9 torch allocations made first thing in the process (what bench.py does)
  synth       the generator's own tensors (carved from its freed temporaries)
  recycled    9 allocations made after 4 GiB of temporaries were allocated and freed
  pages:k     one allocation, stream j at j * (111 + k) 2 MiB pages: k = 1 puts every stream's
              page at the same index mod 8 (TLB-set aliasing, if the set index is the page
              number mod 8), k = 0 / 2 / 3 do not
    python tools/k2_placement.py"""
import ctypes
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import cannikin_synth as synth  # noqa: E402
import paper_2402_05302_b200 as ck  # noqa: E402
from paper_2402_05302_b200 import torch_api as ta  # noqa: E402
from k2_vs_pattern import pattern_lib, timed  # noqa: E402

n, N = 8, 110_000_000
PAGE = 2 << 20


def main():
    torch.cuda.set_device(0)
    virgin = [torch.empty(N, dtype=torch.bfloat16, device="cuda") for _ in range(n + 1)]
    P = pattern_lib()
    b = list(range(1, n + 1))
    r = [x / sum(b) for x in b]
    ctx = ck.Context(world=1, device=0)
    st = torch.zeros(n + 1, dtype=torch.float64, device="cuda")
    nbytes = (n + 1) * N * 2

    def case(tag, bufs):
        gs, out = bufs[:n], bufs[n]
        ptrs = (ctypes.c_void_p * n)(*[g.data_ptr() for g in gs])
        ms_k2 = timed(lambda: ta.weighted_sum_local(ctx, gs, r, out, st[:n], st[n:]))

        def pat():
            P.pattern_launch(ptrs, n, out.data_ptr(), N * 2, 592,
                             ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        ms_p = timed(pat)
        print(json.dumps({"placement": tag, "k2_ms": round(ms_k2, 4),
                          "k2_GBs": round(nbytes / ms_k2 / 1e6, 1), "pattern_ms": round(ms_p, 4),
                          "pattern_GBs": round(nbytes / ms_p / 1e6, 1),
                          "va_page_mod8": [(t.data_ptr() // PAGE) % 8 for t in bufs],
                          "va_offset_mod_page": [t.data_ptr() % PAGE for t in bufs][:3]}),
              flush=True)

    for t in virgin:
        t.normal_()
    case("virgin", virgin)
    if os.environ.get("DATA_ONLY"):
        import numpy as np

        def fill(tag, draw):
            for j, t in enumerate(virgin[:n]):
                t.copy_(draw(j).to(torch.bfloat16))
            case(tag, virgin)

        def fresh(seed_of):
            def d(j):
                g = torch.Generator(device="cuda")
                g.manual_seed(seed_of(j))
                return torch.randn(N, generator=g, device="cuda", dtype=torch.float32)
            return d
        fill("(a) fresh generator per stream, seeds 1000003 + 1009 (j+1) [current recipe]",
             fresh(lambda j: 1000003 + 1009 * (j + 1)))
        ss = np.random.SeedSequence(1).spawn(n)
        fill("(d) fresh generator per stream, SeedSequence.spawn 63-bit seeds",
             fresh(lambda j: int(ss[j].generate_state(1, np.uint64)[0] >> np.uint64(1))))
        g1 = torch.Generator(device="cuda")
        g1.manual_seed(1)
        fill("(b) one generator, streams drawn in sequence",
             lambda j: torch.randn(N, generator=g1, device="cuda", dtype=torch.float32))

        def off(j):
            g = torch.Generator(device="cuda")
            g.manual_seed(1)
            g.set_offset(j * (1 << 32))
            return torch.randn(N, generator=g, device="cuda", dtype=torch.float32)
        fill("(c) one seed, stream j at Philox offset j * 2^32", off)
        fill("(e) fresh generator per stream, seeds j+1", fresh(lambda j: j + 1))
        for t in virgin:
            t.normal_()
        case("normal_ from the default generator", virgin)
        return
    gs = synth.device_gns_gradients(n, N, b, seed=1, dtype="bf16")
    case("synth", gs + [torch.empty_like(gs[0])])
    del gs
    torch.cuda.empty_cache()
    tmp = [torch.empty(1 << 30, dtype=torch.float32, device="cuda") for _ in range(1)]
    del tmp
    recycled = [torch.empty(N, dtype=torch.bfloat16, device="cuda").normal_() for _ in range(n + 1)]
    case("recycled", recycled)
    del recycled
    torch.cuda.empty_cache()
    pages = (N * 2 + PAGE - 1) // PAGE  # 105
    for k in (6, 7, 8, 9, 10, 11):  # stride = pages + k -> 111..116 pages; 112 = 0 mod 8
        stride_pages = pages + k
        big = torch.empty(stride_pages * PAGE * (n + 1) // 2, dtype=torch.bfloat16, device="cuda").normal_()
        per = stride_pages * PAGE // 2
        bufs = [big[j * per: j * per + N] for j in range(n + 1)]
        case(f"pages:{stride_pages}", bufs)
        del bufs, big
        torch.cuda.empty_cache()
    case("virgin_again", virgin)
    # the same buffers with other contents: the inputs of record (bench.py), zeros, normal(0, 1e-3)
    for t, x in zip(virgin, synth.device_gns_gradients(n, N, b, seed=1, dtype="bf16")):
        t.copy_(x)
    torch.cuda.empty_cache()
    case("virgin+synth_data", virgin)
    for t in virgin:
        t.zero_()
    case("virgin+zeros", virgin)
    for t in virgin:
        t.normal_(0.0, 1e-3)
    case("virgin+normal_1e-3", virgin)
    for t in virgin:
        t.normal_()
    case("virgin+normal_1", virgin)


if __name__ == "__main__":
    main()
