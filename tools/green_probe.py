#!/usr/bin/env python
"""Probe: do torch green contexts (SM partitions) cap real compute on this box?  Times a bf16
matmul and a ResNet-18 forward+backward on a green-context stream with 148 / 60 / 40 SMs."""
import json
import sys

import torch
import torchvision
from torch.cuda.green_contexts import GreenContext


def timed(fn, stream, reps=10):
    with torch.cuda.stream(stream):
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    dev = 0
    torch.cuda.set_device(dev)
    a = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
    m = torchvision.models.resnet18(num_classes=10).cuda()
    x = torch.randn(128, 3, 32, 32, device="cuda")

    def mm():
        return a @ a

    # the bench's step_vs_ddp compute: 48 samples x 512 tokens, width 2048
    h = torch.randn(48 * 512, 2048, device="cuda", dtype=torch.bfloat16)
    w = torch.randn(2048, 2048, device="cuda", dtype=torch.bfloat16)
    o = torch.empty_like(h)

    def stack():
        for _ in range(9):
            torch.matmul(h, w, out=o)

    def rn():
        m(x).sum().backward()

    for nsm in [int(v) for v in (sys.argv[1:] or ["148", "60", "40", "16"])]:
        try:
            gc = GreenContext.create(nsm, dev)
            s = gc.Stream()
        except Exception as e:  # noqa: BLE001
            print(json.dumps({"num_sms": nsm, "error": str(e)[:200]}), flush=True)
            continue
        print(json.dumps({"num_sms": nsm, "matmul_ms": round(timed(mm, s), 3),
                          "bench_stack_ms": round(timed(stack, s), 3),
                          "resnet18_b128_fwdbwd_ms": round(timed(rn, s), 3)}), flush=True)
    print(json.dumps({"default_stream": True, "matmul_ms": round(timed(mm, torch.cuda.current_stream()), 3),
                      "resnet18_b128_fwdbwd_ms": round(timed(rn, torch.cuda.current_stream()), 3)}))


if __name__ == "__main__":
    main()
