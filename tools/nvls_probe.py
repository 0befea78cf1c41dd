"""Probe: does this box support multicast (NVLS) memory through torch symmetric memory, and does
NCCL use NVLS?  torchrun --nproc-per-node N tools/nvls_probe.py"""
import os

import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm_mem


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
    try:
        print("backend", symm_mem.get_backend(torch.device("cuda", rank)), flush=True)
    except Exception as e:
        print("backend?", e)
    t = symm_mem.empty(1 << 20, dtype=torch.float32, device=f"cuda:{rank}")
    h = symm_mem.rendezvous(t, dist.group.WORLD.group_name)
    print(rank, "multicast_ptr", hex(h.multicast_ptr), "buffer_ptrs", [hex(p) for p in h.buffer_ptrs],
          "signal_pad_ptrs", [hex(p) for p in h.signal_pad_ptrs][:2], "signal_pad_size",
          symm_mem.get_signal_pad_size(), flush=True)
    x = torch.ones(1 << 24, device="cuda")
    dist.all_reduce(x)
    torch.cuda.synchronize()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
