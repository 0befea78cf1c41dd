"""PyTorch DDP integration: a communication hook that replaces DDP's
per-bucket average with Cannikin's weighted all-reduce g = sum_i r_i g_i (Eq. 9)
and collects the GNS norm statistics of every bucket in the same pass (Eq. 10 inputs).

DDP already does the bucketing and overlaps each bucket's sync with the rest of backprop (the
mechanism §3.2.3 models); the hook only swaps the reduction.  Each rank's local loss
must be the MEAN over its b_i samples (Eq. 1) and r_i = b_i / B.  After backward,
`state.gns_stats()` returns |g_j|^2 for every rank and |g|^2 of the whole gradient (ordered after
the hook's reductions, whatever stream the training loop runs on).

    ctx = torch_api.init_distributed_context(heap_bytes, gated=True)   # gated entry: see below
    state = CannikinHookState(ctx, r_i)
    ddp_model.register_comm_hook(state, cannikin_hook)

The reductions run on the hook's own stream, overlapped with backprop.  Under heterogeneous ranks
a fast rank reaches a bucket before its slow peers; a reduction kernel that waited for them on the
device would hold its CTAs' SMs while the rank's own backward needs them.  With the gated entry
(CANNIKIN_INIT_GATED_ENTRY) that wait is done by a one-warp gate kernel and the reduction grid
only launches once every peer has arrived (bench.py step_vs_ddp: 17.8% saved with the gate, -0.3%
with a 24-CTA grid and no gate, -22% with a full grid and no gate).  DDP's buckets
(25 MB by default) fall in the LL128 kernel's range, which reads and writes only the local bucket
(no staging); larger buckets outside the ctx heap are staged through it.
Argument marshalling only: the reduction runs in libcannikin.so.
"""
import torch

from . import Context
from . import torch_api as ta


class CannikinHookState:
    def __init__(self, ctx: Context, r_i: float, timing: bool = False):
        self.ctx = ctx
        self.r_i = float(r_i)
        self.buckets = 0
        # reductions run on their own stream so they overlap the rest of backprop (§3.2.3)
        self.stream = torch.cuda.Stream(device=torch.device("cuda", ctx.device))
        # optional telemetry for the measured-model loop: per bucket a pair of CUDA
        # events around the reduction (the first one also marks "first bucket ready", Eq. 4)
        self.timing = timing
        self.events = []

    def set_ratio(self, r_i: float):
        """Update r_i = b_i / B when the split changes (a new epoch's plan)."""
        self.r_i = float(r_i)

    def gns_stats(self):
        """Read and reset the statistics of every bucket reduced since the last call: ordered on
        the hook's stream after the calling stream's work (hence after DDP's last bucket)."""
        self.stream.wait_stream(torch.cuda.current_stream())
        return self.ctx.gns_stats(stream=self.stream)


def cannikin_hook(state: CannikinHookState, bucket) -> torch.futures.Future[torch.Tensor]:
    buf = bucket.buffer()
    cs = state.stream
    cs.wait_stream(torch.cuda.current_stream())  # this bucket's gradients are complete
    with torch.cuda.stream(cs):
        if state.timing:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(cs)
        ta.weighted_allreduce(state.ctx, buf, state.r_i, stream=cs)
        if state.timing:
            e1.record(cs)
            state.events.append((e0, e1))
        state.buckets += 1
        # CUDA-aware future: DDP's consumer stream waits for the comm stream, not the host
        fut = torch.futures.Future(devices=[buf.device])
        fut.set_result(buf)
    return fut
