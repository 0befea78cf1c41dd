#!/usr/bin/env python
"""BASELINE configs[1] end to end: ResNet-18 (11,689,512 parameters = the C2 gradient) trained on
synthetic CIFAR-10-shaped data under torch DDP, ranks made heterogeneous, equal-split DDP vs
Cannikin (DDP comm hook + the measured-model loop).

    torchrun --nproc-per-node N tools/ddp_step.py [--B 256 --epochs 4 --iters 10]

Heterogeneity: rank i behaves like a GPU f_i times slower than a B200 (f from Table 1's FP16 TFLOPS,
P:97-99, cyclic A100/V100/P100).  Its real forward and backward are stretched by (f_i - 1) x their
calibrated real durations, injected as K7 delays at the 6 stage boundaries of the network (forward:
after each stage; backward: an identity autograd function per stage), so the buckets of a slow rank
become ready proportionally later, as on a slower GPU.
  DDP:      b_i = B/n, the stock NCCL average.
  Cannikin: the comm hook (weighted all-reduce + norm statistics); every rank measures a_i, P_i,
            gamma_i (first bucket ready / P_i), T_o,i, T_u,i with CUDA events; the analyzer plans
            epoch 0 even, epoch 1 Eq. 8, then OptPerf.
With --hetero sm the ranks are made heterogeneous by SM caps instead (BASELINE north_star:
"per-rank compute-rate caps (restricted grid or SM-partitioned contexts)"): rank i runs its whole
forward/backward/optimizer on the stream of a CUDA green context holding SM_CAPS[mix_i] SMs
(A100 148, V100 60, P100 40: Table 1's FP16 TFLOPS ratios); no injected delays. The
communication (our K3 on the hook's stream, NCCL for DDP) runs in the primary context.
Rank 0 prints one JSON line per epoch and a summary; step times are max over ranks.
"""
import contextlib
import argparse
import json
import os
import statistics
import sys

import torch
import torch.distributed as dist
import torch.nn as nn
import torchvision

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2402_05302_b200 as ck  # noqa: E402
from paper_2402_05302_b200 import torch_api as ta  # noqa: E402
from paper_2402_05302_b200.ddp_hook import CannikinHookState, cannikin_hook  # noqa: E402

NSTAGE = 6
SM_CAPS = {"A100": 148, "V100": 60, "P100": 40}  # 148 x TFLOPS ratio, rounded


class _Delay(torch.autograd.Function):
    """Identity; its backward spends `box[0]` seconds of emulated compute first, and the stage-0
    instance (the last backward op) records `box[1]` = end of backprop compute."""

    @staticmethod
    def forward(ctx, x, box, last):
        ctx.box, ctx.last = box, last
        return x.view_as(x)

    @staticmethod
    def backward(ctx, g):
        if ctx.box[0] > 0:
            ck.emulate_compute(ctx.box[0])
        if ctx.last and ctx.box[1] is not None:
            ctx.box[1].record()
        return g, None, None


class SlowResNet(nn.Module):
    """ResNet-18 with per-stage forward/backward delays (seconds in self.fwd[0], self.bwd[0])."""

    def __init__(self, arch="resnet18", classes=10):
        super().__init__()
        # GroupNorm: per-sample normalisation, valid for any local batch (BatchNorm needs b_i > 1)
        r = getattr(torchvision.models, arch)(num_classes=classes,
                                              norm_layer=lambda c: nn.GroupNorm(8, c))
        self.stages = nn.ModuleList([nn.Sequential(r.conv1, r.bn1, r.relu, r.maxpool), r.layer1,
                                     r.layer2, r.layer3, r.layer4,
                                     nn.Sequential(r.avgpool, nn.Flatten(), r.fc)])
        self.fwd = [0.0]
        self.bwd = [0.0, None]

    def forward(self, x):
        for i, st in enumerate(self.stages):
            if i == 0 and not x.requires_grad:
                x = x.requires_grad_()  # so that the stage-0 backward hook runs
            x = _Delay.apply(x, self.bwd, i == 0)
            x = st(x)
            if self.fwd[0] > 0:
                ck.emulate_compute(self.fwd[0])
        return x


def main():
    os.environ.setdefault("CANNIKIN_SPIN_TIMEOUT_MS", "120000")  # report, do not hang
    ap = argparse.ArgumentParser()
    ap.add_argument("--B", type=int, default=512)
    ap.add_argument("--epochs", type=int, default=4)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--grid", type=int, default=0, help="reduction CTAs (0 = one per SM)")
    ap.add_argument("--ungated", action="store_true",
                    help="wait for late peers inside the reduction grid (no gate kernel)")
    ap.add_argument("--model", default="resnet18", choices=["resnet18", "resnet50"])
    ap.add_argument("--img", type=int, default=32)
    ap.add_argument("--hetero", default="delay", choices=["delay", "sm"])
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    lr = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(lr)
    dist.init_process_group("nccl", device_id=torch.device("cuda", lr))
    torch.backends.cudnn.benchmark = True
    gpu = bench.MIX[rank % len(bench.MIX)]
    f = bench.TFLOPS["A100"] / bench.TFLOPS[gpu]
    if args.hetero == "sm":
        from torch.cuda.green_contexts import GreenContext
        gctx = GreenContext.create(SM_CAPS[gpu], lr)
        cstream = gctx.Stream()
        f = 1.0  # no injected delays: the SM cap is the heterogeneity
        compute = lambda: torch.cuda.stream(cstream)  # noqa: E731
    else:
        compute = contextlib.nullcontext
    B = args.B
    ce = nn.CrossEntropyLoss()
    E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    gen = torch.Generator(device="cuda").manual_seed(1 + rank)
    classes = 10 if args.model == "resnet18" else 1000
    Xall = torch.randn(B, 3, args.img, args.img, device="cuda", generator=gen)
    yall = torch.randint(0, classes, (B,), device="cuda", generator=gen)

    # ---- calibrate this rank's real forward/backward time (no DDP, no delay) vs batch size
    torch.manual_seed(0)
    cal = SlowResNet(args.model, classes).cuda()
    xs, fa, fp = [], [], []
    for bb in (8, 16, 32, 64, 96):
        bb = min(bb, B)
        for rep in range(4):
            with compute():
                e0, e1, e2 = E(), E(), E()
                cal.bwd[1] = None
                e0.record()
                loss = ce(cal(Xall[:bb].clone()), yall[:bb])
                e1.record()
                loss.backward()
                e2.record()
                torch.cuda.synchronize()
                if rep >= 1:
                    xs.append(bb)
                    fa.append(e0.elapsed_time(e1) * 1e-3)
                    fp.append(e1.elapsed_time(e2) * 1e-3)
    qa, sa = ck.fit_linear(xs, fa)
    kp, mp = ck.fit_linear(xs, fp)
    del cal

    def set_slowdown(model, b_i):
        model.fwd[0] = max(0.0, (f - 1.0) * (qa * b_i + sa) / NSTAGE)
        model.bwd[0] = max(0.0, (f - 1.0) * (kp * b_i + mp) / NSTAGE)

    def build(state):
        torch.manual_seed(0)
        m = SlowResNet(args.model, classes).cuda()
        ddp = nn.parallel.DistributedDataParallel(m, device_ids=[lr])
        if state is not None:
            ddp.register_comm_hook(state, cannikin_hook)
        return m, ddp, torch.optim.SGD(ddp.parameters(), lr=0.01, momentum=0.9)

    def run_iter(ddp, model, opt, b_i, state=None):
        with compute():
            return _run_iter(ddp, model, opt, b_i, state)

    def _run_iter(ddp, model, opt, b_i, state=None):
        X, y = Xall[:b_i].clone(), yall[:b_i]
        e0, e1, e2, e3 = E(), E(), E(), E()
        model.bwd[1] = e2  # recorded at the end of backprop compute (before DDP's final wait)
        if state is not None:
            state.events = []
        e0.record()
        loss = ce(ddp(X), y)
        e1.record()
        loss.backward()
        opt.step()
        opt.zero_grad(set_to_none=True)
        e3.record()
        torch.cuda.synchronize()
        return e0, e1, e2, e3

    out = {"model": args.model, "img": args.img,
           "params": sum(p.numel() for p in SlowResNet(args.model, classes).parameters()),
           "mix": [bench.MIX[i % len(bench.MIX)] for i in range(world)], "B": B,
           "calibrated_ms_per_sample": round((qa + kp) * 1e3, 4), "hetero": args.hetero}
    per = [None] * world
    dist.all_gather_object(per, round((qa + kp) * 1e3, 4))
    out["ms_per_sample_by_rank"] = per
    if args.hetero == "sm":
        out["sm_caps"] = [SM_CAPS[bench.MIX[i % len(bench.MIX)]] for i in range(world)]
    # ---------------- equal-split DDP, stock NCCL average
    model, ddp, opt = build(None)
    b_eq = [B // world + (1 if i < B % world else 0) for i in range(world)]
    set_slowdown(model, b_eq[rank])
    steps = []
    for it in range(args.iters + 3):
        dist.barrier()
        e0, e1, e2, e3 = run_iter(ddp, model, opt, b_eq[rank])
        if it >= 3:
            steps.append(e0.elapsed_time(e3))
    t = torch.tensor([statistics.median(steps)], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    out["ddp_ms"] = round(float(t.item()), 3)
    out["b_ddp"] = b_eq
    del ddp, opt, model

    # ---------------- Cannikin: comm hook + measured-model loop
    # gated entry: the wait for a slower peer is done by a one-warp gate kernel, not by the
    # reduction grid (which would take the SMs of this rank's backward pass)
    # DDP's first iteration reduces the whole gradient as one bucket: heap = gradient bytes
    ctx = ta.init_distributed_context(heap_bytes=out["params"] * 4 + (1 << 20), grid=args.grid,
                                      gated=not args.ungated)
    state = CannikinHookState(ctx, 1.0 / world, timing=True)
    model, ddp, opt = build(state)
    an = ck.Analyzer(world)
    gid = 0
    epochs = []
    for epoch in range(args.epochs):
        plan = an.plan(B)
        b = plan["b"]
        state.set_ratio(b[rank] / sum(b))
        set_slowdown(model, b[rank])
        steps = []
        for it in range(args.iters + 2):
            dist.barrier()
            e0, e1, e2, e3 = run_iter(ddp, model, opt, b[rank], state)
            ctx.gns_stats()
            ev = state.events
            a_t = e0.elapsed_time(e1) * 1e-3
            P_t = e1.elapsed_time(e2) * 1e-3
            gam = e1.elapsed_time(ev[0][0]) * 1e-3 / P_t if ev else 0.0
            t_o = sum(x.elapsed_time(y) for x, y in ev[:-1]) * 1e-3
            t_u = ev[-1][0].elapsed_time(ev[-1][1]) * 1e-3 if ev else 0.0
            mine = [a_t, P_t, min(max(gam, 0.0), 0.99), t_o, t_u, e0.elapsed_time(e3)]
            allv = [None] * world
            dist.all_gather_object(allv, mine)
            if it < 2:
                continue
            for node in range(world):
                av, Pv, gv, tov, tuv, _ = allv[node]
                an.observe(node, gid, b[node], av, Pv, gv, tov, tuv)
            gid += 1
            steps.append(max(v[5] for v in allv))
        ep = {"epoch": epoch, "phase": plan["phase"], "b": b,
              "measured_ms": round(statistics.median(steps), 3),
              "predicted_ms": None if plan["T_pred"] != plan["T_pred"] else round(plan["T_pred"] * 1e3, 3)}
        epochs.append(ep)
        if rank == 0:
            print(json.dumps(ep), flush=True)
    out["cannikin_ms"] = epochs[-1]["measured_ms"]
    out["b_cannikin"] = epochs[-1]["b"]
    out["saving"] = round(1 - out["cannikin_ms"] / out["ddp_ms"], 4)
    out["predicted_ms"] = epochs[-1]["predicted_ms"]
    if out["predicted_ms"]:
        out["prediction_error"] = round(abs(out["predicted_ms"] - out["cannikin_ms"]) / out["cannikin_ms"], 4)
    out["buckets_per_step"] = len(state.events)
    out["k3_grid"] = args.grid
    out["gated_entry"] = not args.ungated
    if rank == 0:
        print(json.dumps({"summary": out}), flush=True)
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
