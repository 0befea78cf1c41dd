"""torch.Tensor conveniences over the C ABI (argument marshalling only).

PyTorch supplies device memory, streams and process groups; every step of the hot path runs in
libcannikin.so.
"""
from __future__ import annotations

import torch

from . import BF16, F32, Context, get_unique_id
from . import weighted_allreduce_group as _group_ar

_CODES = {torch.float32: F32, torch.bfloat16: BF16}


def dtype_code(dt: torch.dtype) -> int:
    if dt not in _CODES:
        raise TypeError(f"cannikin supports float32 and bfloat16 gradients, not {dt}")
    return _CODES[dt]


class _DeviceView:
    """Expose a raw device pointer owned by a cannikin ctx as a torch tensor (no copy)."""

    def __init__(self, ptr: int, numel: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (numel,), "typestr": typestr,
                                         "data": (ptr, False), "version": 3, "strides": None}


def bucket_tensor(ctx: Context, numel: int, dtype: torch.dtype) -> torch.Tensor:
    """Allocate a peer-mapped bucket from the ctx heap (collective for world > 1) and view it as a
    tensor.  The ctx owns the memory; free it with ``free_bucket_tensor``."""
    esz = torch.empty(0, dtype=dtype).element_size()
    ptr = ctx.alloc_bucket(max(numel * esz, 1))
    typestr = {torch.float32: "<f4", torch.bfloat16: "<i2"}[dtype]
    t = torch.as_tensor(_DeviceView(ptr, numel, typestr), device=f"cuda:{ctx.device}")
    return t.view(dtype) if dtype == torch.bfloat16 else t


def free_bucket_tensor(ctx: Context, t: torch.Tensor):
    ctx.free_bucket(t.data_ptr())


def _cur(stream):
    return stream if stream is not None else torch.cuda.current_stream()


def weighted_allreduce(ctx: Context, bucket: torch.Tensor, r_i: float, stream=None):
    """In place: bucket <- sum_j r_j g_j over all ranks (Eq. 9), norms accumulated in the ctx."""
    assert bucket.is_cuda and bucket.is_contiguous()
    ctx.weighted_allreduce(bucket.data_ptr(), bucket.numel(), dtype_code(bucket.dtype), r_i,
                           _cur(stream))


def gns_stats_bucket(ctx: Context, bucket: torch.Tensor, b_i: int, stream=None):
    """Out-of-place Eq. 10 inputs of one bucket (bucket unchanged): ([|g_j|^2], |g|^2)."""
    assert bucket.is_cuda and bucket.is_contiguous()
    return ctx.gns_stats_bucket(bucket.data_ptr(), bucket.numel(), dtype_code(bucket.dtype), b_i,
                                _cur(stream))


def weighted_allreduce_group(ctxs, buckets, r, stream=None):
    """Every rank of an in-process group (Context.group_local) in ONE kernel launch: buckets[k]
    <- sum_j r[j] buckets[j] (Eq. 9), norms accumulated in every rank's ctx."""
    n, dt = buckets[0].numel(), buckets[0].dtype
    for b in buckets:
        assert b.is_cuda and b.is_contiguous() and b.numel() == n and b.dtype == dt
    _group_ar(ctxs, [b.data_ptr() for b in buckets], n, dtype_code(dt), list(r), _cur(stream))


def weighted_allreduce_nccl(ctx: Context, bucket: torch.Tensor, r_i: float, stream=None):
    """As weighted_allreduce, through NCCL reduce-scatter / all-gather with fused pre/post kernels
    (K4): any device tensor, no peer mapping."""
    assert bucket.is_cuda and bucket.is_contiguous()
    ctx.weighted_allreduce_nccl(bucket.data_ptr(), bucket.numel(), dtype_code(bucket.dtype), r_i,
                                _cur(stream))


def weighted_sum_local(ctx: Context, grads, r, out: torch.Tensor, local_sq: torch.Tensor,
                       global_sq: torch.Tensor, accumulate: bool = False, stream=None,
                       variant=None, chain: bool = False):
    """Emulated ranks on one GPU: out <- sum_j r_j grads[j]; local_sq[j] <- |grads[j]|^2;
    global_sq <- |out|^2 (float64 device tensors).  chain=True: consecutive bucket of the same
    gradient (its inputs are not produced by the kernel just before; CANNIKIN_LOCAL_CHAIN)."""
    dt = dtype_code(out.dtype)
    # local_sq / global_sq: float64 device tensors or pinned (device-mapped) host tensors
    for g in grads:
        assert g.is_cuda and g.is_contiguous() and g.dtype == out.dtype and g.numel() == out.numel()
    assert local_sq.dtype == torch.float64 and global_sq.dtype == torch.float64
    ctx.weighted_sum_local([g.data_ptr() for g in grads], list(r), out.data_ptr(), out.numel(), dt,
                           local_sq.data_ptr(), global_sq.data_ptr(), accumulate, _cur(stream),
                           variant, chain)


def ddp_allreduce_mean(ctx: Context, bucket: torch.Tensor, stream=None):
    ctx.ddp_allreduce_mean(bucket.data_ptr(), bucket.numel(), dtype_code(bucket.dtype), _cur(stream))


def init_distributed_context(heap_bytes: int, grid: int = 0, group=None,
                             check_ratios: bool = False, gated: bool = False) -> Context:
    """Create the ctx of this rank of an initialised torch.distributed group: rank 0 draws the NCCL
    unique id, which is broadcast over the torch process group (plumbing only)."""
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    obj = [get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    dev = torch.cuda.current_device()
    return Context(rank=rank, world=world, unique_id=obj[0], device=dev, heap_bytes=heap_bytes,
                   grid=grid, check_ratios=check_ratios, gated=gated)


class McBucket:
    """A symmetric, multicast-capable bucket from torch symmetric memory (device-memory plumbing)
    for cannikin_weighted_allreduce_nvls.  `tensor` is this rank's copy."""

    def __init__(self, numel: int, dtype: torch.dtype, group=None):
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem

        self.tensor = symm_mem.empty(numel, dtype=dtype, device=torch.cuda.current_device())
        g = group if group is not None else dist.group.WORLD
        self.handle = symm_mem.rendezvous(self.tensor, g.group_name)
        self.mc_ptr = int(self.handle.multicast_ptr)
        if not self.mc_ptr:
            raise RuntimeError("multicast (NVLS) memory is not available on this system")


def weighted_allreduce_nvls(ctx: Context, mcb: "McBucket", r_i: float, view=None, stream=None):
    """In place over mcb.tensor (or a slice `view` of it): Eq. 9 through NVSwitch multicast."""
    t = mcb.tensor if view is None else view
    off = t.data_ptr() - mcb.tensor.data_ptr()
    ctx.weighted_allreduce_nvls(t.data_ptr(), mcb.mc_ptr + off, t.numel(), dtype_code(t.dtype),
                                r_i, _cur(stream))
