"""Per-rank worker for tests/test_gpu_ddp.py: ResNet-18 (GroupNorm, so every sample's loss is
independent and Eq. 9's equivalence with the full-batch mean is exact) under torch DDP with the
Cannikin comm hook, uneven local batches.  Saves the rank's averaged gradient, a full-batch
single-process reference gradient, the local gradient's norm and the hook's statistics."""
import argparse
import copy
import os
import sys

import numpy as np
import torch
import torch.distributed as dist
import torch.nn as nn
import torchvision

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2402_05302_b200 import torch_api as ta  # noqa: E402
from paper_2402_05302_b200.ddp_hook import CannikinHookState, cannikin_hook  # noqa: E402


def flat_grad(model):
    return torch.cat([p.grad.reshape(-1) for p in model.parameters()])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    lr = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(lr)
    dist.init_process_group("nccl", device_id=torch.device("cuda", lr))
    torch.backends.cudnn.deterministic = True
    torch.backends.cudnn.benchmark = False
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.manual_seed(0)
    model = torchvision.models.resnet18(num_classes=10,
                                        norm_layer=lambda c: nn.GroupNorm(8, c)).cuda()
    ref_model = copy.deepcopy(model)
    loc_model = copy.deepcopy(model)
    b = [17, 9, 23, 5, 11, 30, 2, 7][:world]
    B = sum(b)
    g = torch.Generator(device="cuda").manual_seed(123)
    X = torch.randn(B, 3, 32, 32, device="cuda", generator=g)
    y = torch.randint(0, 10, (B,), device="cuda", generator=g)
    lo = sum(b[:rank])
    Xl, yl = X[lo:lo + b[rank]], y[lo:lo + b[rank]]
    ce = nn.CrossEntropyLoss()  # mean over the batch: local loss = mean over b_i samples (Eq. 1)
    # full-batch reference: mean over all B samples
    ce(ref_model(X), y).backward()
    ref = flat_grad(ref_model)
    # this rank's local gradient g_i (for |g_i|^2)
    ce(loc_model(Xl), yl).backward()
    gi = flat_grad(loc_model)
    ctx = ta.init_distributed_context(heap_bytes=64 << 20, gated=True)  # as ddp_hook.py documents
    ddp = nn.parallel.DistributedDataParallel(model, device_ids=[lr], bucket_cap_mb=4)
    state = CannikinHookState(ctx, b[rank] / B)
    ddp.register_comm_hook(state, cannikin_hook)
    # iteration 1 (DDP builds its buckets), then iteration 2 on the rebuilt buckets
    ce(ddp(Xl), yl).backward()
    torch.cuda.synchronize()
    ctx.gns_stats()
    model.zero_grad(set_to_none=False)
    state.buckets = 0
    ce(ddp(Xl), yl).backward()
    torch.cuda.synchronize()
    got = flat_grad(model)
    loc, glob = ctx.gns_stats()
    # a third iteration read through the hook state's own ordering (no host synchronisation
    # between backward and the read: state.gns_stats() orders itself after DDP's last bucket)
    model.zero_grad(set_to_none=False)
    ce(ddp(Xl), yl).backward()
    hloc, hglob = state.gns_stats()
    np.savez(os.path.join(args.out, f"rank{rank}.npz"), got=got.cpu().numpy(), ref=ref.cpu().numpy(),
             gi=gi.cpu().numpy(), gi_sq=float((gi.double() ** 2).sum()), loc=np.array(loc),
             glob=glob, buckets=state.buckets, hook_loc=np.array(hloc), hook_glob=hglob,
             b=np.array(b))
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
