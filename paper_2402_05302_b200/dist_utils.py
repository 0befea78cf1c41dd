"""Host-side plumbing for the multi-process path (one process per GPU, torch.distributed).

Nothing here touches gradients: the device work is in libcannikin.so.  These helpers are what
every rank runs around it -- distributing the NCCL unique id, the replicated per-step control
logic (GNS estimate + OptPerf split from identical inputs, so no collective is needed for them,
SURVEY §3 CS2/CS4) and max-over-ranks timing.  They work with any backend (gloo on CPU for tests).
"""
from __future__ import annotations

from typing import Callable

import torch
import torch.distributed as dist

from . import gns_estimate, opt_split


def broadcast_unique_id(make_id: Callable[[], bytes], group=None) -> bytes:
    """Rank 0 calls make_id() (cannikin_get_unique_id); the 128 bytes go to every rank."""
    obj = [make_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    uid = obj[0]
    assert isinstance(uid, (bytes, bytearray)) and len(uid) == 128
    return bytes(uid)


def max_over_ranks(x: float, device="cpu", group=None) -> float:
    """The multi-rank time of a step is the slowest rank's (contract: max over ranks)."""
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def control_step(local_sq, global_sq, b, models, comm, B_next):
    """The host half of one step, replicated on every rank: heterogeneous GNS estimate from the
    norm statistics (bitwise identical on all ranks) and the split for the next step."""
    est = gns_estimate(local_sq, global_sq, b) if len(b) >= 2 else None
    split = opt_split(models, comm, B_next)
    return est, split
