#!/usr/bin/env python
"""The paper's closed loop on B200: learn the per-node models from measured timings and reach
OptPerf "as early as the third epoch", with the prediction error of §5.3.

    torchrun --nproc-per-node N tools/optperf_loop.py [--epochs 5 --iters 6 --B 96]

Every rank runs its emulated compute (K7, the Eq. 3 model of its GPU class, as in bench.py's
step comparison) and the real weighted all-reduce (K3) of the C4 gradient in 9 buckets overlapped
with the emulated backprop.  Each iteration every rank measures, with CUDA events, its a_i, P_i,
gamma_i (first-bucket share of backprop), T_o_i and T_u_i (its sync times, including any wait for
slower ranks); the observations are all-gathered and fed to the analyzer on every rank
(cannikin_analyzer_*), which plans the next epoch: even split, Eq. 8, then OptPerf.  Rank 0
prints one JSON line per epoch: plan, measured step time (max over ranks), predicted time.
"""
import argparse
import json
import os
import statistics
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import cannikin_synth as synth  # noqa: E402
import paper_2402_05302_b200 as ck  # noqa: E402
from paper_2402_05302_b200 import torch_api as ta  # noqa: E402


def main():
    os.environ.setdefault("CANNIKIN_SPIN_TIMEOUT_MS", "120000")  # report, do not hang
    ap = argparse.ArgumentParser()
    ap.add_argument("--epochs", type=int, default=5)
    ap.add_argument("--iters", type=int, default=6)
    ap.add_argument("--B", type=int, default=96)
    ap.add_argument("--N", type=int, default=110_000_000)
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    lr = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(lr)
    dist.init_process_group("nccl", device_id=torch.device("cuda", lr))
    N, NB = args.N, 9
    ctx = ta.init_distributed_context(heap_bytes=N * 2)
    bucket = ta.bucket_tensor(ctx, N, torch.bfloat16)
    bucket.copy_(synth.device_gns_gradients(world, N, [1] * world, seed=0, dtype="bf16",
                                            ranks=[rank])[0])
    be = (N // NB) - (N // NB) % 8
    cuts = [i * be for i in range(NB)] + [N]
    models = bench.hetero_models(world)
    q, s0, k, m = models[rank]
    cs, ms = torch.cuda.current_stream(), torch.cuda.Stream()
    an = ck.Analyzer(world)
    E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    it = 0
    for epoch in range(args.epochs):
        plan = an.plan(args.B)
        b = plan["b"]
        r = b[rank] / sum(b)
        times = []
        for i in range(args.iters + 1):  # the first iteration of an epoch is a warm-up
            dist.barrier()
            torch.cuda.synchronize()
            e_start, e_fwd = E(), E()
            e_chunk = [E() for _ in range(NB)]
            c_beg = [E() for _ in range(NB)]
            c_end = [E() for _ in range(NB)]
            e_start.record(cs)
            ck.emulate_compute(q * b[rank] + s0, cs)
            e_fwd.record(cs)
            for j in range(NB):
                ck.emulate_compute((k * b[rank] + m) / NB, cs)
                e_chunk[j].record(cs)
                ms.wait_event(e_chunk[j])
                c_beg[j].record(ms)
                ta.weighted_allreduce(ctx, bucket[cuts[j]:cuts[j + 1]], r, stream=ms)
                c_end[j].record(ms)
            cs.wait_stream(ms)
            e_stop = E()
            e_stop.record(cs)
            torch.cuda.synchronize()
            ctx.gns_stats(cs)
            a_t = e_start.elapsed_time(e_fwd) * 1e-3
            P_t = e_fwd.elapsed_time(e_chunk[-1]) * 1e-3
            gam = e_fwd.elapsed_time(e_chunk[0]) * 1e-3 / P_t
            # sync times as this node sees them: from its bucket being ready to the sync's end
            t_o = sum(e_chunk[j].elapsed_time(c_end[j]) for j in range(NB - 1)) * 1e-3
            t_u = e_chunk[-1].elapsed_time(c_end[-1]) * 1e-3
            step = e_start.elapsed_time(e_stop) * 1e-3
            mine = [a_t, P_t, gam, t_o, t_u, step]
            allv = [None] * world
            dist.all_gather_object(allv, mine)
            if i == 0:
                continue
            for node in range(world):
                av, Pv, gv, tov, tuv, _ = allv[node]
                an.observe(node, it, b[node], av, Pv, gv, tov, tuv)
            times.append(max(v[5] for v in allv))
            it += 1
        meas = statistics.median(times)
        if rank == 0:
            out = {"epoch": epoch, "phase": plan["phase"], "b": b, "measured_ms": round(meas * 1e3, 4),
                   "predicted_ms": None if plan["T_pred"] != plan["T_pred"] else round(plan["T_pred"] * 1e3, 4),
                   "mix": [bench.MIX[i % len(bench.MIX)] for i in range(world)]}
            if out["predicted_ms"] is not None:
                out["prediction_error"] = round(abs(out["predicted_ms"] - out["measured_ms"]) / out["measured_ms"], 4)
            print(json.dumps(out), flush=True)
    if rank == 0:
        nodes, comm = an.models()
        opt = ck.opt_split(models, comm, args.B)
        print(json.dumps({"learned_models": nodes, "true_models": models, "learned_comm": comm,
                          "opt_split_true_models": opt["b"]}), flush=True)
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
