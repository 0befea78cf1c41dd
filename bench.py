#!/usr/bin/env python
"""Benchmark of the Cannikin data-parallel hot path on B200 (one JSON line on rank 0).

A *step* is one pass of the whole hot path over one batch of synthetic gradients:
  weighted aggregation g = sum_i r_i g_i with the fused norms |g_i|^2, |g|^2   (Eq. 9-10)
  -> read the norm statistics -> heterogeneous GNS estimate (Theorem 1)
  -> OptPerf split for the next step (opt_split).
N = 1 : the ranks are emulated on one GPU (K2, `cannikin_weighted_sum_local`); with --bucket-mb
        the gradient is cut into buckets whose K2 launches are PDL-chained.
N > 1 : one process per GPU (torchrun); `cannikin_weighted_allreduce` (K3 variants over NVLink).
value : gradient bytes aggregated per second, n x N x s per step (n ranks, emulated at N = 1) --
        the same quantity at every N.  The roofline object uses each bound's own bytes: K2's HBM
        bytes (n+1) N s at N = 1, the bus bytes 2(n-1)/n N s per rank at N > 1.

    python bench.py [--gpus N --steps K --warmup W --config c4 --impl {cannikin,reference}]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# ---------------------------------------------------------------------------- workloads
# Gradient sizes from the paper's Table 4; 355M is BASELINE.json's sweep model.
CONFIGS = {
    "c1": {"workload": "c1: 3 emulated heterogeneous ranks, 2^20 fp32 gradient, b={32,64,96}",
           "N": 1 << 20, "dtype": "f32", "n_emu": 3, "B": 192, "fixed_b": [32, 64, 96]},
    "c2": {"workload": "c2: ResNet-18/CIFAR-10 gradient, 11,689,512 fp32, unequal b_i",
           "N": 11_689_512, "dtype": "f32", "n_emu": 2, "B": 64, "fixed_b": [24, 40]},
    "c3": {"workload": "c3: ResNet-50/ImageNet gradient, 25,557,032 fp32, P100/V100/A100 mix",
           "N": 25_557_032, "dtype": "f32", "n_emu": 8, "B": 400},
    "c4": {"workload": "c4: BERT-base SQuAD gradient, 110,000,000 bf16, P100/V100/A100 mix",
           "N": 110_000_000, "dtype": "bf16", "n_emu": 8, "B": 96},
    "c5": {"workload": "c5: 355M-param gradient, 354,823,168 fp32, P100/V100/A100 mix",
           "N": 354_823_168, "dtype": "f32", "n_emu": 8, "B": 400},
}

# Heterogeneous node models (Eq. 3) with per-sample speed in the ratio of Table 1's
# FP16 TFLOPS (A100 77.97, V100 31.4, P100 21.2) -- the C3/C4 emulated mix.
TFLOPS = {"A100": 77.97, "V100": 31.4, "P100": 21.2}
# cyclic so that every prefix is heterogeneous; the 8-rank mix is C3's 3 A100 / 3 V100 / 2 P100
MIX = ["A100", "V100", "P100", "A100", "V100", "P100", "A100", "V100"]
COMM = (0.20, 0.010, 0.004)  # gamma, T_o, T_u


def node_models(n):
    out = []
    for i in range(n):
        f = TFLOPS["A100"] / TFLOPS[MIX[i % len(MIX)]]
        out.append((0.0004 * f, 0.004, 0.0008 * f, 0.002))  # q, s, k, m  (seconds)
    return out


def hetero_models(n):
    """Per-node (q, s, k, m) in seconds for the emulated-compute tools (tools/optperf_loop.py,
    tools/adaptive_batch.py): an A100-class node spends 0.04 ms/sample forward and 0.08 ms/sample
    backward (+0.3 / 0.2 ms fixed); slower nodes scale the per-sample terms by Table 1's TFLOPS
    ratio."""
    out = []
    for i in range(n):
        f = TFLOPS["A100"] / TFLOPS[MIX[i % len(MIX)]]
        out.append((0.04e-3 * f, 0.3e-3, 0.08e-3 * f, 0.2e-3))
    return out


# Compute-rate caps for the step-time comparison (north_star: "per-rank compute-rate caps (...
# SM-partitioned contexts)"): rank i runs its compute on a CUDA green context holding this many of
# the 148 SMs -- 148 x Table 1's FP16 TFLOPS ratio A100 : V100 : P100, rounded.
SM_CAPS = {"A100": 148, "V100": 60, "P100": 40}


def hetero_sm_compare(N, s, tdt, rank, world, local_rank, B, iters, dist, ta, ck, torch,
                      grid=0, gated=True):
    """Step time of Cannikin against equal-split DDP on ranks made heterogeneous by REAL compute
    under SM caps (green contexts, SM_CAPS by the cyclic A100/V100/P100 mix), not by injected
    delays.  The compute is a synthetic layer stack of bf16 GEMMs (each sample = T tokens of width
    H; forward NB GEMMs, backward NB chunks of two GEMMs), so its time is linear in b_i at a rate
    the SM cap sets.  Bucket j of the C4 gradient (NB buckets) is reduced on a comm stream as soon
    as backward chunk j is done (§3.2.3 overlap).  Cannikin: the measured-model loop --
    epoch 0 even split, epoch 1 Eq. 8, epoch 2 OptPerf from the models the analyzer LEARNED from
    per-rank CUDA-event timings (a_i, P_i, gamma_i, T_o, T_u) -- with the fused weighted
    all-reduce.  DDP: b_i = B/n with the NCCL average.  The prediction error compares the
    analyzer's Eq. 7 prediction with the measured step.  Max over ranks throughout.
    `gated` (CANNIKIN_INIT_GATED_ENTRY): a fast rank waits for its slow peers in a one-warp gate
    kernel instead of in the reduction grid, which would otherwise hold SMs its own backward pass
    needs; `grid` is the reduction kernels' CTA count (0 = one per SM)."""
    from torch.cuda.green_contexts import GreenContext

    NB, T, H = 9, 512, 2048
    gpu = MIX[rank % len(MIX)]
    gctx = GreenContext.create(SM_CAPS[gpu], local_rank)
    cs = gctx.Stream()
    ms = torch.cuda.Stream()
    ctx = ta.init_distributed_context(heap_bytes=N * s, grid=grid, gated=gated)
    bucket = ta.bucket_tensor(ctx, N, tdt)
    bucket.normal_()
    cuts = [j * (N // NB - (N // NB) % 8) for j in range(NB)] + [N]
    gen = torch.Generator(device="cuda").manual_seed(7)
    Wt = [torch.randn(H, H, device="cuda", dtype=torch.bfloat16, generator=gen) * 0.02
          for _ in range(NB)]
    acts = [torch.randn(B * T, H, device="cuda", dtype=torch.bfloat16, generator=gen) * 0.1
            for _ in range(NB + 1)]
    dx = torch.empty(B * T, H, device="cuda", dtype=torch.bfloat16)
    dw = [torch.empty(H, H, device="cuda", dtype=torch.bfloat16) for _ in range(NB)]
    stats = torch.zeros(world + 1, dtype=torch.float64, device="cuda")
    E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    ev = [(E(), E(), E()) for _ in range(NB)]  # (chunk done, comm start, comm end)

    def step(b_i, r_i, ours):
        M = b_i * T
        e0, e1, e2, e3 = E(), E(), E(), E()
        with torch.cuda.stream(cs):
            e0.record(cs)
            for l in range(NB):
                torch.matmul(acts[l][:M], Wt[l], out=acts[l + 1][:M])
            e1.record(cs)
            for j in range(NB):
                l = NB - 1 - j
                torch.matmul(acts[l + 1][:M], Wt[l].t(), out=dx[:M])
                torch.matmul(acts[l][:M].t(), acts[l + 1][:M], out=dw[l])
                ev[j][0].record(cs)
                ms.wait_event(ev[j][0])
                with torch.cuda.stream(ms):
                    ev[j][1].record(ms)
                    if ours:
                        ta.weighted_allreduce(ctx, bucket[cuts[j]:cuts[j + 1]], r_i, stream=ms)
                    else:
                        ta.ddp_allreduce_mean(ctx, bucket[cuts[j]:cuts[j + 1]], stream=ms)
                    ev[j][2].record(ms)
            e2.record(cs)
            cs.wait_stream(ms)
            if ours:
                ctx.gns_stats_async(stats.data_ptr(), cs)
            e3.record(cs)
        torch.cuda.synchronize()
        a_t = e0.elapsed_time(e1) * 1e-3
        P_t = e1.elapsed_time(e2) * 1e-3
        gam = e1.elapsed_time(ev[0][0]) * 1e-3 / P_t
        t_o = sum(ev[j][1].elapsed_time(ev[j][2]) for j in range(NB - 1)) * 1e-3
        t_u = ev[NB - 1][1].elapsed_time(ev[NB - 1][2]) * 1e-3
        return [a_t, P_t, min(max(gam, 0.0), 0.99), t_o, t_u, e0.elapsed_time(e3)]

    def run(b_vec, ours, count, an=None, gid0=0):
        steps = []
        for it in range(count + 2):
            dist.barrier()
            mine = step(b_vec[rank], b_vec[rank] / sum(b_vec), ours)
            allv = [None] * world
            dist.all_gather_object(allv, mine)  # plumbing: every rank's timings, off the clock
            if it < 2:
                continue
            if an is not None:
                for node in range(world):
                    an.observe(node, gid0 + it, b_vec[node], *allv[node][:5])
            steps.append(max(v[5] for v in allv))
        return statistics.median(steps)

    b_eq = [B // world + (1 if i < B % world else 0) for i in range(world)]
    ddp_ms = run(b_eq, False, iters)
    an = ck.Analyzer(world)
    epochs = []
    for ep in range(3):
        plan = an.plan(B)
        meas = run(plan["b"], True, iters, an, 100 * ep)
        epochs.append({"epoch": ep, "phase": plan["phase"], "b": plan["b"],
                       "measured_ms": round(meas, 4),
                       "predicted_ms": None if plan["T_pred"] != plan["T_pred"]
                       else round(plan["T_pred"] * 1e3, 4)})
    nodes, comm = an.models()
    last = epochs[-1]
    out = {"cannikin_ms": last["measured_ms"], "ddp_ms": round(ddp_ms, 4),
           "saving": round(1.0 - last["measured_ms"] / ddp_ms, 4),
           "predicted_cannikin_ms": last["predicted_ms"],
           "prediction_error": (None if last["predicted_ms"] is None else
                                round(abs(last["predicted_ms"] - last["measured_ms"])
                                      / last["measured_ms"], 4)),
           "b_cannikin": last["b"], "b_ddp": b_eq, "epochs": epochs, "buckets": NB,
           "mix": [MIX[i % len(MIX)] for i in range(world)],
           "sm_caps": [SM_CAPS[MIX[i % len(MIX)]] for i in range(world)],
           "learned_ms_per_sample": [round((q + k) * 1e3, 4) for q, _, k, _ in nodes],
           "learned_comm": {"gamma": round(comm[0], 4), "t_o_ms": round(comm[1] * 1e3, 4),
                            "t_u_ms": round(comm[2] * 1e3, 4)},
           "compute": f"bf16 GEMM stack, {T} tokens x {H} wide per sample, {NB} layers",
           "reduction": {"gated_entry": gated, "grid": grid or "one CTA per SM"},
           "note": "heterogeneity = real compute on SM-capped green contexts; split from models "
                   "learned from measured timings (not from the generator); comm kernels real; "
                   "median step of the last epoch, max over ranks"}
    ta.free_bucket_tensor(ctx, bucket)
    ctx.close()
    return out


# One GPU shared by heterogeneous tenants (the paper's Cluster C shares GPUs among jobs,
# P:603-608): disjoint SM partitions in Table 1's A100 : V100 : P100 proportion, rounded
# to the 8-SM granularity of sm_100 green contexts, a few SMs left to the reduction.
SHARED_GPU_MIX = ["A100", "V100", "P100"]
SHARED_GPU_SMS = [[80, 32, 24], [64, 24, 16], [48, 16, 16]]  # the first the device can split


def hetero_shared_gpu(ctx, N, tdt, B, iters, ta, ck, torch):
    """Step time of Cannikin against equal-split DDP for 3 ranks sharing ONE GPU on disjoint SM
    partitions (cannikin_green_partitions), real compute, no injected delays: the single-GPU
    counterpart of hetero_sm_compare.  Rank i runs a synthetic bf16 GEMM stack (each sample = T
    tokens of width H; forward NB GEMMs, backward NB chunks of two GEMMs) on its partition's stream;
    bucket j of the C4 gradient is reduced by K2 over the three ranks' buckets on a comm stream as
    soon as every rank's backward chunk j is done (§3.2.3 overlap).  Cannikin: the
    measured-model loop (epoch 0 even split, epoch 1 Eq. 8, epoch 2 OptPerf from models the analyzer
    LEARNED from per-rank CUDA-event timings), K2 with r_i = b_i / B; DDP: b_i = B/n, K2
    with r_i = 1/n (the mean, Eq. 2).  Prediction error: the analyzer's Eq. 7 prediction against
    the measured step."""
    import statistics

    n, NB, T, H = len(SHARED_GPU_MIX), 9, 512, 2048
    green, errs = None, []
    for counts in SHARED_GPU_SMS:
        try:
            green = ck.GreenPartitions(counts, device=torch.cuda.current_device())
            break
        except ck.CannikinError as e:
            errs.append(str(e))
    if green is None:
        raise RuntimeError("; ".join(errs))
    try:
        rs = [torch.cuda.ExternalStream(h) for h in green.streams]
        cs = torch.cuda.Stream()
        master = torch.cuda.current_stream()
        gen = torch.Generator(device="cuda").manual_seed(7)
        Wt = [torch.randn(H, H, device="cuda", dtype=torch.bfloat16, generator=gen) * 0.02
              for _ in range(NB)]
        acts = [[torch.randn(B * T, H, device="cuda", dtype=torch.bfloat16, generator=gen) * 0.1
                 for _ in range(NB + 1)] for _ in range(n)]
        dx = [torch.empty(B * T, H, device="cuda", dtype=torch.bfloat16) for _ in range(n)]
        dw = [[torch.empty(H, H, device="cuda", dtype=torch.bfloat16) for _ in range(NB)]
              for _ in range(n)]
        grads = [torch.randn(N, device="cuda", dtype=torch.float32, generator=gen).to(tdt)
                 for _ in range(n)]
        out = torch.empty(N, device="cuda", dtype=tdt)
        st = torch.zeros(n + 1, dtype=torch.float64, device="cuda")
        cuts = [j * (N // NB - (N // NB) % 8) for j in range(NB)] + [N]
        E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

        def step(b, r):
            t0, t9 = E(), E()
            fw = [(E(), E()) for _ in range(n)]  # forward start / end per rank
            ch = [[E() for _ in range(NB)] for _ in range(n)]  # backward chunk j done per rank
            cm = [(E(), E()) for _ in range(NB)]  # reduction of bucket j start / end
            t0.record(master)
            for i in range(n):
                rs[i].wait_stream(master)
                with torch.cuda.stream(rs[i]):
                    M = b[i] * T
                    fw[i][0].record(rs[i])
                    for l in range(NB):
                        torch.matmul(acts[i][l][:M], Wt[l], out=acts[i][l + 1][:M])
                    fw[i][1].record(rs[i])
                    for j in range(NB):
                        l = NB - 1 - j
                        torch.matmul(acts[i][l + 1][:M], Wt[l].t(), out=dx[i][:M])
                        torch.matmul(acts[i][l][:M].t(), acts[i][l + 1][:M], out=dw[i][l])
                        ch[i][j].record(rs[i])
            for j in range(NB):
                for i in range(n):
                    cs.wait_event(ch[i][j])
                a, c = cuts[j], cuts[j + 1]
                cm[j][0].record(cs)
                ta.weighted_sum_local(ctx, [g[a:c] for g in grads], r, out[a:c], st[:n], st[n:],
                                      accumulate=j > 0, stream=cs)
                cm[j][1].record(cs)
            for i in range(n):
                master.wait_stream(rs[i])
            master.wait_stream(cs)
            t9.record(master)
            torch.cuda.synchronize()
            t_o = sum(cm[j][0].elapsed_time(cm[j][1]) for j in range(NB - 1)) * 1e-3
            t_u = cm[NB - 1][0].elapsed_time(cm[NB - 1][1]) * 1e-3
            per_rank = []
            for i in range(n):
                a_t = fw[i][0].elapsed_time(fw[i][1]) * 1e-3
                P_t = fw[i][1].elapsed_time(ch[i][NB - 1]) * 1e-3
                gam = fw[i][1].elapsed_time(ch[i][0]) * 1e-3 / P_t
                per_rank.append((a_t, P_t, min(max(gam, 0.0), 0.99), t_o, t_u))
            return per_rank, t0.elapsed_time(t9)

        def run(b, r, count, an=None, gid0=0):
            steps = []
            for it in range(count + 2):
                per_rank, ms = step(b, r)
                if it < 2:
                    continue
                if an is not None:
                    for i in range(n):
                        an.observe(i, gid0 + it, b[i], *per_rank[i])
                steps.append(ms)
            return statistics.median(steps)

        b_eq = [B // n + (1 if i < B % n else 0) for i in range(n)]
        ddp_ms = run(b_eq, [1.0 / n] * n, iters)
        an = ck.Analyzer(n)
        epochs = []
        for ep in range(3):
            plan = an.plan(B)
            meas = run(plan["b"], [x / B for x in plan["b"]], iters, an, 100 * ep)
            epochs.append({"epoch": ep, "phase": plan["phase"], "b": plan["b"],
                           "measured_ms": round(meas, 4),
                           "predicted_ms": None if plan["T_pred"] != plan["T_pred"]
                           else round(plan["T_pred"] * 1e3, 4)})
        nodes, comm = an.models()
        last = epochs[-1]
        return {"cannikin_ms": last["measured_ms"], "ddp_ms": round(ddp_ms, 4),
                "saving": round(1.0 - last["measured_ms"] / ddp_ms, 4),
                "predicted_cannikin_ms": last["predicted_ms"],
                "prediction_error": (None if last["predicted_ms"] is None else
                                     round(abs(last["predicted_ms"] - last["measured_ms"])
                                           / last["measured_ms"], 4)),
                "b_cannikin": last["b"], "b_ddp": b_eq, "epochs": epochs, "buckets": NB,
                "mix": SHARED_GPU_MIX, "sm_partitions": green.sms,
                "partition_attempts_refused": errs,
                "learned_ms_per_sample": [round((q + k) * 1e3, 4) for q, _, k, _ in nodes],
                "learned_comm": {"gamma": round(comm[0], 4), "t_o_ms": round(comm[1] * 1e3, 4),
                                 "t_u_ms": round(comm[2] * 1e3, 4)},
                "compute": f"bf16 GEMM stack, {T} tokens x {H} wide per sample, {NB} layers",
                "note": "3 ranks sharing one GPU on disjoint SM partitions (green contexts; "
                        "Cluster C, P:603-608), real compute, split from models learned from "
                        "measured timings; reduction = K2 over the ranks' buckets; median step of "
                        "the last epoch"}
    finally:
        torch.cuda.synchronize()
        green.close()


# C4's "adaptive global batch via GNS" (BASELINE configs[3]): candidate total batches, B0 = 9
ADAPTIVE_CANDS = [9, 16, 32, 64, 96, 128, 192, 256, 384, 512, 768, 1024]


def adaptive_batch_sidecar(ctx, N, n, epochs, steps, synth, ck, ta, torch, rank=0, world=1,
                           bucket=None):
    """The paper's outer loop on the bench gradient (one GPU, n emulated ranks, K2): the true noise
    scale trS/|G|^2 rises 50 -> 5000 over the epochs (the shape of fig:gns); every step
    the ranks' mean gradients for their b_i are drawn from the V1 recipe, K2 reduces them and
    returns the norms, the library estimates G and S (Theorem 1) and updates the EMA (reading Q26);
    at the end of each epoch the total batch is chosen by goodput (reading Q27) and split
    by opt_split.  Reports per epoch B, the split, the true and estimated B_noise.  world > 1: one
    rank per GPU, each draws its own mean gradient into the heap bucket and K3 reduces it (the
    statistics, hence every estimate and every choice, are identical on all ranks)."""
    models = hetero_models(n)
    comm = (1.0 / 9, 8 * 65e-6, 65e-6)
    if world == 1:
        out = torch.empty(N, dtype=torch.bfloat16, device="cuda")
        st = torch.zeros(n + 1, dtype=torch.float64, device="cuda")
    ema = ck.GnsEma(0.9)
    B = max(ADAPTIVE_CANDS[0], n)
    rows = []
    errs_t1, errs_cor = [], []
    for e in range(epochs):
        trS = 50.0 * (100.0 ** (e / max(1, epochs - 1)))
        split = ck.opt_split(models, comm, B)["b"]
        for k in range(steps):
            if world == 1:
                gs = synth.device_gns_gradients(n, N, split, G2=1.0, trS=trS, seed=1000 * e + k,
                                                dtype="bf16")
                ta.weighted_sum_local(ctx, gs, [x / B for x in split], out, st[:n], st[n:])
                v = st.tolist()
            else:
                gs = synth.device_gns_gradients(n, N, split, G2=1.0, trS=trS, seed=1000 * e + k,
                                                dtype="bf16", ranks=[rank])
                bucket.copy_(gs[0])
                ta.weighted_allreduce(ctx, bucket, split[rank] / B)
                loc, glob = ctx.gns_stats()
                v = list(loc) + [glob]
            est = ck.gns_estimate(v[:n], v[n], split)
            cor = ck.gns_estimate(v[:n], v[n], split, corrected=True)  # §8(f)-4, reading Q31
            errs_t1.append(abs(est["B_noise"] - trS) / trS)
            errs_cor.append(abs(cor["B_noise"] - trS) / trS)
            ema.update(est["G2"], est["trS"])
            del gs
        nxt = ck.choose_batch(models, comm, ADAPTIVE_CANDS, ADAPTIVE_CANDS[0], ema.B_noise)
        rows.append({"epoch": e, "B": B, "split": split, "true_B_noise": round(trS, 1),
                     "est_B_noise": round(est["B_noise"], 1), "ema_B_noise": round(ema.B_noise, 1),
                     "next_B": nxt["B"]})
        B = nxt["B"]
    torch.cuda.empty_cache()
    last_err = max(abs(r["est_B_noise"] - r["true_B_noise"]) / r["true_B_noise"] for r in rows)
    return {"epochs": rows, "B_path": [r["B"] for r in rows] + [B],
            "max_rel_err_last_step_B_noise": round(last_err, 4),
            "mean_rel_err_B_noise": {"theorem1": round(sum(errs_t1) / len(errs_t1), 5),
                                     "corrected_weights": round(sum(errs_cor) / len(errs_cor), 5),
                                     "steps": len(errs_t1)},
            "note": "synthetic noise-scale schedule 50 -> 5000; B chosen by goodput from the EMA "
                    "of the Theorem-1 estimates computed from the K2 statistics"}


def bucketed_sidecar(launch, N, s, n, world, bucket_mb, steps, peak, alg_bytes, dist, torch):
    """The paper's bucketed regime (DDP-style buckets) on the bench gradient: the step's
    reduction cut into buckets of `bucket_mb` per rank, one library call per bucket, captured in
    one CUDA graph and timed as a chain (first start to last end, CUDA events, max over ranks).
    launch(a, c, first) enqueues the call for elements [a, c).  At N = 1 consecutive K2 launches are
    PDL-chained (CANNIKIN_LOCAL_CHAIN), so a launch's duration is the chain's / launches."""
    be = int(bucket_mb * 2**20) // s
    be -= be % 8
    cuts = list(range(0, N, be)) + [N]
    nb = len(cuts) - 1

    def seq():
        for i in range(nb):
            launch(cuts[i], cuts[i + 1], i == 0)

    seq()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        seq()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / steps], device="cuda", dtype=torch.float64)
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    chain_ms = float(t.item())
    out = {"bucket_mb": bucket_mb, "launches_per_step": nb, "chain_ms": round(chain_ms, 4),
           "kernel_ms": round(chain_ms / nb, 4),
           "value": round(n * N * s / (chain_ms * 1e-3) / 1e9, 2), "unit": "GB/s"}
    if world == 1:
        ach = alg_bytes / (chain_ms * 1e-3) / 1e9
        out["roofline"] = {"bound": "hbm", "achieved": round(ach, 1), "peak": peak,
                           "frac": round(ach / peak, 4),
                           "kernel": "wsum_local_kernel (K2), PDL-chained bucket launches"}
    else:
        busbw = N * s / (chain_ms * 1e-3) * 2 * (n - 1) / n / 1e9
        out["roofline"] = {"bound": "nvlink", "achieved": round(busbw, 1), "peak": 770.0,
                           "frac": round(busbw / 770.0, 4),
                           "nominal_frac": round(busbw / 900.0, 4)}
    return out


def nvls_sidecar(ctx, N, rank, world, r_i, steps, dist, ta, torch):
    """fp32 weighted all-reduce of N elements through NVSwitch multicast (K6) next to the two-shot
    kernel (K3) on the same bytes: kernel time (CUDA events, max over ranks) and busbw."""
    s = 4
    mcb = ta.McBucket(N, torch.float32)
    mcb.tensor.normal_()
    res = {"elements": N, "dtype": "f32"}

    def timed(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / steps], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    t6 = timed(lambda: ta.weighted_allreduce_nvls(ctx, mcb, r_i))
    ctx.gns_stats()
    res["k6_ms"] = round(t6, 4)
    res["k6_busbw"] = round(N * s / (t6 * 1e-3) * 2 * (world - 1) / world / 1e9, 1)
    res["note"] = ("NVLS moves ~(1+1/n) N s per direction vs the two-shot's 2(n-1)/n N s, plus a "
                   "local scaling pass; fp32 only")
    del mcb
    return res


def k4_sidecar(ctx, bucket, N, s, r_i, world, steps, barrier, stream, dist, ta, torch):
    """cannikin_weighted_allreduce_nccl (K4) on the bench bucket: kernel-path time, max over ranks."""
    for _ in range(3):
        ta.weighted_allreduce_nccl(ctx, bucket, r_i)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        ta.weighted_allreduce_nccl(ctx, bucket, r_i)
    e1.record(stream)
    barrier()
    km = torch.tensor([e0.elapsed_time(e1) / steps], device="cuda", dtype=torch.float64)
    dist.all_reduce(km, op=dist.ReduceOp.MAX)
    ctx.gns_stats()
    k4ms = float(km.item())
    return {"ms": round(k4ms, 4),
            "busbw": round(N * s / (k4ms * 1e-3) * 2 * (world - 1) / world / 1e9, 1),
            "note": "cannikin_weighted_allreduce_nccl: fp32 pre-kernel + ncclReduceScatter + "
                    "post-kernel + ncclAllGather, same bucket, statistics included"}


def esize(dtype):
    return 4 if dtype == "f32" else 2


# ---------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons DURING the timed region (B200_PROFILING.md)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,clocks.mem")

    def __init__(self, device: int):
        self.device, self.lines, self.proc = device, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms",
                 "100", "-i", str(self.device)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.25)
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        sm, mem, mx, reasons = [], [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 6:
                continue
            try:
                sm.append(float(p[0]))
                mx = float(p[1])
            except ValueError:
                continue
            for nm, v in zip(names, p[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
            if len(p) > 6:
                try:
                    mem.append(float(p[6]))
                except ValueError:
                    pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "mem_mhz": statistics.median(mem) if mem else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# SM-driven peer writes with every GPU sending to every peer at once, per direction (GB/s):
# profiles/r01/nvlink_bw_n2.jsonl (write2), nvlink_bw_n4.jsonl (a2a_write4); 8 GPUs not measured
BIDIR_WRITE_GBS = {2: 690.8, 4: 671.4}


def pattern_ceiling(gs, out, N, s, achieved, ck, torch):
    """The bare memory pattern of K2 (cannikin_probe_stream_pattern: the same n + 1 streams of
    16-byte vectors, integer adds, no arithmetic of the method) timed on the bench's own buffers
    right after the timed region -- the HBM ceiling K2's traffic can reach in this run's memory
    state; best of three grids, back-to-back launches, CUDA events."""
    try:
        ptrs = [g.data_ptr() for g in gs]
        nbytes = N * s // 16 * 16
        tried = {}
        for cps in (3, 4, 5):
            for _ in range(3):
                ck.probe_stream_pattern(ptrs, out.data_ptr(), nbytes, cps)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                ck.probe_stream_pattern(ptrs, out.data_ptr(), nbytes, cps)
            e1.record()
            torch.cuda.synchronize()
            tried[f"{cps}_ctas_per_sm"] = round((len(gs) + 1) * nbytes / (e0.elapsed_time(e1) / 10 * 1e-3) / 1e9, 1)
        best = max(tried.values())
        return {"peak": best, "frac": round(achieved / best, 4), "tried": tried,
                "kind": "live bare n:1 stream pattern on the same buffers after the timed region "
                        "(cannikin_probe_stream_pattern), best of three grids"}
    except Exception as e:  # noqa: BLE001
        return {"unavailable": str(e)[:200]}


def a2a_ceiling(ctx, heap_bytes, n, steps, busbw, barrier, stream, dist, torch):
    """The all-to-all peer-write ceiling of this box at this N, measured live with
    cannikin_probe_a2a_write (every rank writes heap/n bytes into every peer at once; per-direction
    GB/s = (n-1) x bytes / time, max over ranks); falls back to the earlier tools/nvlink_bw.cu
    figures if the probe is unavailable."""
    try:
        per = (heap_bytes // n) // 16 * 16
        rep = max(1, (1 << 30) // ((n - 1) * per))  # >= 1 GiB of egress per launch
        best, tried = 0.0, {}
        for cps in (1, 2, 4):  # the ceiling is the best of three launch shapes
            for _ in range(2):
                ctx.probe_a2a_write(per, rep, cps, stream.cuda_stream)
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = max(3, min(steps, 10))
            e0.record(stream)
            for _ in range(reps):
                ctx.probe_a2a_write(per, rep, cps, stream.cuda_stream)
            e1.record(stream)
            barrier()
            t = torch.tensor([e0.elapsed_time(e1) / reps], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            gbs = (n - 1) * per * rep / (float(t.item()) * 1e-3) / 1e9
            tried[f"{cps}_ctas_per_sm"] = round(gbs, 1)
            best = max(best, gbs)
        return {"peak": round(best, 1), "frac": round(busbw / best, 4), "tried": tried,
                "kind": f"live {n}-GPU all-to-all peer writes per direction "
                        f"(cannikin_probe_a2a_write, {per >> 20} MiB per peer x {rep}, "
                        "best launch shape, this run): a plain SM copy of the all-to-all "
                        "pattern, which K3's fused protocol can exceed (W = 4)"}
    except Exception as e:  # noqa: BLE001
        if n not in BIDIR_WRITE_GBS:
            return {"unavailable": str(e)[:200]}
        return {"peak": BIDIR_WRITE_GBS[n], "frac": round(busbw / BIDIR_WRITE_GBS[n], 4),
                "kind": f"earlier {n}-GPU all-to-all write probe (tools/nvlink_bw.cu)"}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except (OSError, ValueError):
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def ncu_traffic(tag):
    """dram bytes per launch of the dominant kernel from the committed ncu --set full summary."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f)
        v = d.get(tag)
        return float(v) if isinstance(v, (int, float)) else None
    except (OSError, ValueError):
        return None


# ---------------------------------------------------------------------------- CPU oracle legs
def oracle_step(gs, r, dtype, b, models, B):
    """One oracle pass over a bounded sample: Eq. 9 + norms, GNS estimate, split."""
    from oracle import aggregate as agg
    from oracle import gns as ogns
    from oracle import optsplit as osp

    g, ls, gsq = agg.aggregate(gs, r, dtype)
    if len(b) >= 2:
        ogns.gns_estimate(ls, gsq, b)
    osp.int_split_greedy(models, COMM, B)
    return g


def cpu_sample(cfg, n, sample_elems, seed=0):
    import cannikin_synth as synth
    from oracle import aggregate as agg

    b = cfg.get("fixed_b") or [max(1, cfg["B"] // n)] * n
    b = (b * n)[:n]
    gs = synth.gns_gradients(n, sample_elems, b, seed=seed, dtype=cfg["dtype"])
    return gs, agg.ratios(b), b


def cpu_baseline(cfg, n, seconds=10.0, sample_elems=1 << 22):
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    gs, r, b = cpu_sample(cfg, n, sample_elems)
    models = node_models(n)
    calls, t0 = 0, time.perf_counter()
    while True:
        oracle_step(gs, r, cfg["dtype"], b, models, cfg["B"])
        calls += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    nbytes = n * sample_elems * esize(cfg["dtype"])  # the metric: gradient bytes aggregated
    out = {"value": round(nbytes * calls / el / 1e9, 4), "unit": "GB/s", "cores": 1,
           "kind": "oracle",
           "sample": f"{calls} oracle passes over {n} ranks x {sample_elems} {cfg['dtype']} "
                     f"elements (first 2^22 of the workload shape), {el:.1f} s, numpy float64 "
                     "single-threaded"}
    out["all_cores"] = cpu_baseline_all_cores(cfg, n, gs, r)
    return out


def _oracle_chunk_worker(args):
    """One process: the oracle's Eq. 9 + norms over a fixed chunk, repeated for `seconds`."""
    gs, r, dtype, seconds = args
    os.environ["OMP_NUM_THREADS"] = "1"
    from oracle import aggregate as agg

    calls, t0 = 0, time.perf_counter()
    while True:
        agg.aggregate(gs, r, dtype)
        calls += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            return calls, el


def cpu_baseline_all_cores(cfg, n, gs, r, seconds=5.0, chunk=1 << 18):
    """SURVEY §8(d) oracle timing (b): the same oracle over fixed chunks on every host core at
    once (one process per core, chunk boundaries fixed, results identical); GB/s summed."""
    import multiprocessing as mp

    cores = max(1, min(os.cpu_count() or 1, 128))
    N = len(gs[0])
    bounds = [(a, min(a + chunk, N)) for a in range(0, N, chunk)]
    jobs = [([g[a:c] for g in gs], r, cfg["dtype"], seconds)
            for k, (a, c) in enumerate(bounds * ((cores + len(bounds) - 1) // len(bounds)))][:cores]
    try:
        with mp.get_context("fork").Pool(cores) as pool:
            res = pool.map(_oracle_chunk_worker, jobs)
    except Exception as e:  # noqa: BLE001
        return {"error": str(e)[:200]}
    es = esize(cfg["dtype"])
    gbps = sum(n * len(j[0][0]) * es * c / el for j, (c, el) in zip(jobs, res)) / 1e9
    return {"value": round(gbps, 3), "unit": "GB/s", "cores": cores, "kind": "oracle",
            "sample": f"{cores} processes, each the oracle's Eq. 9 + norms over a fixed "
                      f"{chunk}-element chunk of the same {n}-rank sample for {seconds:.0f} s"}


def run_reference(args, cfg, rank, world):
    """--impl reference: the CPU oracle as it stands, on rank 0 only (others exit 0)."""
    if rank != 0:
        return
    n = cfg["n_emu"] if world == 1 else world
    sample = 1 << 22
    gs, r, b = cpu_sample(cfg, n, sample)
    models = node_models(n)
    for _ in range(args.warmup):
        oracle_step(gs, r, cfg["dtype"], b, models, cfg["B"])
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle_step(gs, r, cfg["dtype"], b, models, cfg["B"])
    el = time.perf_counter() - t0
    nbytes = n * sample * esize(cfg["dtype"])  # the metric: gradient bytes aggregated
    val = nbytes * args.steps / el / 1e9
    line = {"impl": "reference", "metric": "weighted-allreduce+GNS GB/s (% HBM/NVLink roofline)", "value": round(val, 4),
            "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(el / args.steps * 1e3, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["workload"], "emulated_ranks": n,
                       "sample_elements_per_rank": sample},
            "cpu_baseline": {"value": round(val, 4), "unit": "GB/s", "cores": 1, "kind": "oracle",
                             "sample": f"each step: oracle Eq.9+norms over {n} x {sample} "
                                       f"{cfg['dtype']} elements, GNS estimate, opt_split"},
            "e2e": {"value": round(val, 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="cannikin", choices=["cannikin", "reference"])
    ap.add_argument("--n-emulated", type=int, default=0, help="N=1: emulated ranks (0 = config)")
    ap.add_argument("--bucket-mb", type=float, default=0.0, help="bucket size per rank (0 = whole)")
    ap.add_argument("--dtype", default=None, choices=[None, "f32", "bf16"])
    ap.add_argument("--grid", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch eagerly instead of a CUDA graph")
    ap.add_argument("--no-hetero", action="store_true",
                    help="skip the step-time-vs-DDP comparison and the adaptive-batch sidecar")
    ap.add_argument("--hetero-grid", type=int, default=0,
                    help="step-vs-DDP: CTAs of the reduction kernels (0 = one per SM)")
    ap.add_argument("--hetero-ungated", action="store_true",
                    help="step-vs-DDP: wait for late peers inside the reduction grid (no gate)")
    ap.add_argument("--no-nvls", action="store_true", help="skip the NVLS fp32 sidecar")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    cfg = dict(CONFIGS[args.config])
    if args.dtype:
        cfg["dtype"] = args.dtype
    if args.n_emulated:
        cfg["n_emu"] = args.n_emulated

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    # a bench must end: a peer wait longer than 2 min reports a protocol error instead of hanging
    os.environ.setdefault("CANNIKIN_SPIN_TIMEOUT_MS", "120000")
    if args.impl == "reference":
        return run_reference(args, cfg, rank, world)

    import numpy as np
    import torch

    import cannikin_synth as synth
    import paper_2402_05302_b200 as ck
    from paper_2402_05302_b200 import torch_api as ta

    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    tdt = {"f32": torch.float32, "bf16": torch.bfloat16}[cfg["dtype"]]
    N, s = cfg["N"], esize(cfg["dtype"])
    n = cfg["n_emu"] if world == 1 else world
    models = node_models(n)
    split = ck.opt_split(models, COMM, cfg["B"]) if "fixed_b" not in cfg else None
    b = cfg.get("fixed_b") if world == 1 and "fixed_b" in cfg else (split["b"] if split else None)
    if b is None or len(b) != n:
        b = ck.opt_split(models, COMM, max(cfg["B"], n))["b"]
    B = sum(b)
    r = [x / B for x in b]
    bucket_elems = N if args.bucket_mb <= 0 else max(1, int(args.bucket_mb * 2**20) // s)
    bucket_elems -= bucket_elems % 8
    cuts = list(range(0, N, bucket_elems)) + [N]
    peaks, peak_kind = measured_peaks()

    def launches_per_step():
        return len(cuts) - 1

    # two statistics buffers: the host half of step t (GNS estimate, split) runs while the GPU
    # already executes step t+1 -- the paper consumes B_noise and r_opt per epoch, not per step
    NBUF = 2
    stats_h = [torch.empty(n + 1, dtype=torch.float64, pin_memory=True) for _ in range(NBUF)]
    stats_d = [torch.zeros(n + 1, dtype=torch.float64, device="cuda") for _ in range(NBUF)]
    ready = [torch.cuda.Event() for _ in range(NBUF)]
    nb = len(cuts) - 1
    if world == 1:
        ctx = ck.Context(world=1, device=local_rank)
        gs = synth.device_gns_gradients(n, N, b, seed=0, dtype=cfg["dtype"])
        out = torch.empty(N, dtype=tdt, device="cuda")
        alg_bytes = (n + 1) * N * s  # K2's HBM algorithmic bytes (roofline)

        # one bucket: its last CTA writes the n+1 statistics straight into pinned host memory
        # (mapped, device-accessible), no readback copy.  Several buckets: they accumulate in
        # device memory (a host-memory read-modify-write per bucket would sit on the chain's
        # critical path) and one 72-byte copy reads them back.
        st_acc = stats_h if nb == 1 else stats_d

        def launch(bi, k):
            a, c = cuts[bi], cuts[bi + 1]
            # buckets after the first are PDL-chained (CANNIKIN_LOCAL_CHAIN): their loads start
            # while the previous bucket's last CTAs finish
            ta.weighted_sum_local(ctx, [g[a:c] for g in gs], r, out[a:c], st_acc[k][:n],
                                  st_acc[k][n:], accumulate=bi > 0, chain=bi > 0)

        def read_stats(k):
            if nb > 1:
                stats_h[k].copy_(stats_d[k], non_blocking=True)
    else:
        ctx = ta.init_distributed_context(heap_bytes=N * s, grid=args.grid)
        bucket = ta.bucket_tensor(ctx, N, tdt)
        g0 = synth.device_gns_gradients(n, N, b, seed=0, dtype=cfg["dtype"], ranks=[rank])[0]
        bucket.copy_(g0)
        del g0
        alg_bytes = 2 * (n - 1) * N * s  # whole-job NVLink bus bytes, n x 2(n-1)/n N s

        def launch(bi, k):
            a, c = cuts[bi], cuts[bi + 1]
            ta.weighted_allreduce(ctx, bucket[a:c], r[rank])

        def read_stats(k):  # one finalize kernel writes straight into pinned host memory
            ctx.gns_stats_async(stats_h[k].data_ptr(), torch.cuda.current_stream())

    # per-kernel timing events on the launching stream (external: recordable inside a graph)
    evs = [[(torch.cuda.Event(enable_timing=True, external=True),
             torch.cuda.Event(enable_timing=True, external=True)) for _ in range(nb)]
           for _ in range(NBUF)]

    # N = 1 with several buckets: consecutive K2 launches overlap (PDL), so they are timed as one
    # chain (first start to last end) and a launch's duration is the chain's / nb
    chain_timing = world == 1 and nb > 1

    def device_part(k):
        if chain_timing:
            evs[k][0][0].record()
            for bi in range(nb):
                launch(bi, k)
            evs[k][0][1].record()
        else:
            for bi in range(nb):
                evs[k][bi][0].record()
                launch(bi, k)
                evs[k][bi][1].record()
        read_stats(k)

    kernel_ms = []

    # the host half of a step (GNS estimate + EMA + next split) is one native call
    control = ck.ControlStep(b, models, COMM, B)

    def host_part(k, record=False):
        ready[k].synchronize()
        control(stats_h[k].data_ptr())
        if record:
            if chain_timing:
                a, c = evs[k][0]
                kernel_ms.extend([a.elapsed_time(c) / nb] * nb)
            else:
                kernel_ms.extend(a.elapsed_time(c) for a, c in evs[k])

    graphs = None
    for k in range(NBUF):
        device_part(k)
        ready[k].record()
        host_part(k)
    if not args.no_graph:
        # the device half of a step is one CUDA graph (kernels + stats readback): no per-kernel
        # host launch latency
        torch.cuda.synchronize()
        graphs = []
        for k in range(NBUF):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                device_part(k)
            graphs.append(g)
        torch.cuda.synchronize()

    def run_steps(count, record=False):
        for t in range(count):
            k = t % NBUF
            if graphs is not None:
                graphs[k].replay()
            else:
                device_part(k)
            ready[k].record()
            if t > 0:
                host_part((t - 1) % NBUF, record)
        host_part((count - 1) % NBUF, record)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    run_steps(args.warmup)
    # ---- timed region: K steps, events on the launching stream, max over ranks
    stream = torch.cuda.current_stream()
    with ClockSampler(local_rank) as clk:
        barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        run_steps(args.steps, record=True)
        t1.record(stream)
        barrier()
    ms = t0.elapsed_time(t1)
    if dist is not None:
        tt = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
        kk = torch.tensor([statistics.mean(kernel_ms)], device="cuda", dtype=torch.float64)
        dist.all_reduce(kk, op=dist.ReduceOp.MAX)
        kmean = float(kk.item())
    else:
        kmean = statistics.mean(kernel_ms)
    kq = statistics.quantiles(kernel_ms, n=10) if len(kernel_ms) >= 2 else [kmean] * 9
    kdist = {"p10": round(kq[0], 4), "p50": round(statistics.median(kernel_ms), 4),
             "p90": round(kq[8], 4), "launches": len(kernel_ms), "rank": rank}
    ms_step = ms / args.steps
    # value: gradient bytes aggregated per second, n x N x s per step (n = emulated ranks at N = 1,
    # GPUs at N > 1) -- the same quantity at every N; the roofline below uses each bound's bytes
    grad_bytes = n * N * s
    value = grad_bytes / (ms_step * 1e-3) / 1e9

    # ---- roofline of the dominant kernel (per launch)
    launch_bytes = alg_bytes / launches_per_step()
    if world == 1:
        achieved = launch_bytes / (kmean * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"],
                "unit": "GB/s", "frac": round(achieved / peaks["hbm_gbs"], 4),
                "peak_kind": peak_kind,
                "kernel": ("wsum_local_kernel (K2)" if nb == 1 else
                           f"wsum_local_kernel (K2), {nb} PDL-chained bucket launches per step, "
                           "timed as one chain: kernel_ms = chain / launches"),
                "kernel_ms": round(kmean, 4), "kernel_ms_dist": kdist,
                "traffic": ncu_traffic(f"{args.config}_n{n}_{cfg['dtype']}_b{launches_per_step()}"),
                "pattern_ceiling": pattern_ceiling(gs, out, N, s, achieved, ck, torch)}
    else:
        busbw = (N * s / len(cuts[:-1])) / (kmean * 1e-3) * 2 * (n - 1) / n / 1e9
        roof = {"bound": "nvlink", "achieved": round(busbw, 1), "peak": 770.0, "unit": "GB/s",
                "frac": round(busbw / 770.0, 4),
                "peak_kind": "measured peer copy per GPU per direction (B200_PROFILING.md)",
                "nominal": {"peak": 900.0, "frac": round(busbw / 900.0, 4),
                            "kind": "NVLink 5 nominal per GPU per direction (north_star)"},
                "kernel": f"K3 {ctx.last_variant()} (variant chosen by size)",
                "kernel_ms": round(kmean, 4), "kernel_ms_dist": kdist,
                "traffic": ncu_traffic(f"{args.config}_w{n}_{cfg['dtype']}"),
                # an all-reduce loads BOTH directions at once; the same SM-driven copy with both
                # directions busy peaks lower than the one-way 770: measured live, this run
                "bidir_ceiling": a2a_ceiling(ctx, N * s, n, args.steps, busbw, barrier, stream,
                                             dist, torch)}

    # ---- DDP baseline (equal split, NCCL average) on the same bucket, N > 1
    ddp = None
    if world > 1:
        for _ in range(3):
            ta.ddp_allreduce_mean(ctx, bucket)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            ta.ddp_allreduce_mean(ctx, bucket)
        e1.record(stream)
        barrier()
        dm = torch.tensor([e0.elapsed_time(e1) / args.steps], device="cuda", dtype=torch.float64)
        dist.all_reduce(dm, op=dist.ReduceOp.MAX)
        ddp = {"ms_per_allreduce": round(float(dm.item()), 4),
               "note": "ncclAllReduce(avg) of the same bucket, equal-split DDP semantics (Eq. 2)"}

    # ---- the same weighted all-reduce through NCCL reduce-scatter / all-gather (K4), N > 1
    if world > 1:
        try:
            ddp["k4_nccl_path"] = k4_sidecar(ctx, bucket, N, s, r[rank], world, args.steps,
                                             barrier, stream, dist, ta, torch)
        except Exception as e:  # a sidecar must not sink the bench line
            ddp["k4_nccl_path"] = {"unavailable": str(e)[:200]}

    # ---- the bucketed regime (DDP-style 25 MB buckets per rank) next to the whole-gradient line
    bucketed = None
    if nb == 1:
        if world == 1:
            sc = torch.zeros(n + 1, dtype=torch.float64, device="cuda")

            def blaunch(a, c, first):
                ta.weighted_sum_local(ctx, [g[a:c] for g in gs], r, out[a:c], sc[:n], sc[n:],
                                      accumulate=not first, chain=not first)
        else:
            def blaunch(a, c, first):
                ta.weighted_allreduce(ctx, bucket[a:c], r[rank])
        try:
            bucketed = bucketed_sidecar(blaunch, N, s, n, world, 25.0, args.steps,
                                        peaks["hbm_gbs"], alg_bytes, dist, torch)
            if world > 1:
                bucketed["kernel"] = f"K3 {ctx.last_variant()}"
                ctx.gns_stats()
        except Exception as e:  # a sidecar must not sink the bench line
            bucketed = {"unavailable": str(e)[:200]}

    # ---- NVSwitch-multicast (NVLS) variant, fp32 sidecar on the same element count (K6)
    nvls = None
    if world > 1 and not args.no_nvls:
        try:
            nvls = nvls_sidecar(ctx, N, rank, world, r[rank], args.steps, dist, ta, torch)
        except Exception as e:  # multicast unavailable on this system
            nvls = {"unavailable": str(e)[:200]}

    adaptive = None
    if not args.no_hetero and cfg["dtype"] == "bf16":
        try:
            keep = None if world == 1 else bucket.clone()  # the bench bucket, restored after
            adaptive = adaptive_batch_sidecar(ctx, N, n, 6, 3, synth, ck, ta, torch, rank=rank,
                                              world=world, bucket=None if world == 1 else bucket)
            if keep is not None:
                bucket.copy_(keep)
                del keep
        except Exception as e:  # a sidecar must not sink the bench line
            adaptive = {"unavailable": str(e)[:200]}

    hetero = None
    if world == 1 and not args.no_hetero:
        try:
            hetero = hetero_shared_gpu(ctx, N, tdt, cfg["B"], 6, ta, ck, torch)
        except Exception as e:  # green contexts unavailable: report, do not sink the bench line
            hetero = {"unavailable": str(e)[:300]}
    if world > 1 and not args.no_hetero:
        try:
            hetero = hetero_sm_compare(N, s, tdt, rank, world, local_rank, max(B, world), 6, dist,
                                       ta, ck, torch, grid=args.hetero_grid,
                                       gated=not args.hetero_ungated)
        except Exception as e:  # green contexts unavailable: report, do not sink the bench line
            hetero = {"unavailable": str(e)[:300]}

    # ---- end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        if world == 1:
            host = [torch.empty(N, dtype=tdt, pin_memory=True) for _ in range(n)]
            for h, g in zip(host, gs):
                h.copy_(g)
            h2d = n * N * s

            def e2e_step():
                for h, g in zip(host, gs):
                    g.copy_(h, non_blocking=True)
                eager_step()
        else:
            host = torch.empty(N, dtype=tdt, pin_memory=True)
            host.copy_(bucket)
            h2d = N * s

            def e2e_step():
                bucket.copy_(host, non_blocking=True)
                eager_step()
        def eager_step():  # the plain public-API calls a user makes, no graph, no overlap
            for bi in range(nb):
                launch(bi, 0)
            read_stats(0)
            ready[0].record()
            host_part(0)

        d2h = (n + 1) * 8
        ek = max(3, min(args.steps, 10))
        e2e_step()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(ek):
            e2e_step()
        e1.record(stream)
        barrier()
        em = torch.tensor([e0.elapsed_time(e1) / ek], device="cuda", dtype=torch.float64)
        if dist is not None:
            dist.all_reduce(em, op=dist.ReduceOp.MAX)
        em = float(em.item())
        e2e = {"value": round(grad_bytes / (em * 1e-3) / 1e9, 3), "unit": "GB/s",
               "ms_per_step": round(em, 3), "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "steps": ek}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(cfg, n)

    if rank == 0:
        line = {
            "metric": "weighted-allreduce+GNS GB/s (% HBM/NVLink roofline)",
            "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": cfg["dtype"], "data": "synthetic",
            "config": {"workload": cfg["workload"], "elements": N, "ranks": n,
                       "emulated": world == 1, "b": b, "B": B,
                       "buckets_per_step": launches_per_step(),
                       "value_model": "gradient bytes aggregated per second: n*N*s per step "
                                      "(n ranks, emulated at N=1), the same quantity at every N",
                       "grad_bytes_per_step": grad_bytes,
                       "roofline_bytes_per_step": alg_bytes,
                       "roofline_bytes_model": ("(n+1)*N*s HBM (K2)" if world == 1 else
                                                "n*2(n-1)/n*N*s NVLink bus bytes (K3)"),
                       "l2": (f"inputs larger than L2 ({alg_bytes / 126e6:.1f}x 126 MB), no flush"
                              if alg_bytes > 2 * 126e6 else
                              "working set fits in L2 (not flushed): latency-bound case, "
                              "not a roofline claim"),
                       "cuda_graph": graphs is not None,
                       "host_overlap": "host half of step t overlaps device half of step t+1"},
            "roofline": roof, "bucketed_25mb": bucketed, "cpu_baseline": cpu, "e2e": e2e,
            "ddp_baseline": ddp,
            "step_vs_ddp": hetero, "adaptive_batch": adaptive, "nvls_f32": nvls,
            # K2 / K3 per bucket, plus (N > 1) the statistics-finalize kernel per step
            "gpu_launches": (launches_per_step() + (1 if world > 1 else 0)) * args.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        ctx.close()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
