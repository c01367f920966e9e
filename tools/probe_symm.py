"""Probe torch symmetric memory on the GPU box (multicast / peer pointers).
torchrun --nproc-per-node 2 tools/probe_symm.py"""
import os
import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
t = symm.empty(1 << 20, dtype=torch.float32, device="cuda")
h = symm.rendezvous(t, dist.group.WORLD.group_name)
print(rank, "backend", symm.get_backend("cuda") if hasattr(symm, "get_backend") else "?",
      "mc", hex(h.multicast_ptr or 0),
      "peers", [hex(p) for p in h.buffer_ptrs], "sig", h.signal_pad_size,
      "bufsize", h.buffer_size, "offset", getattr(h, "offset", None), flush=True)
t2 = symm.empty(3 << 20, dtype=torch.bfloat16, device="cuda")
h2 = symm.rendezvous(t2, dist.group.WORLD.group_name)
print(rank, "second", hex(t2.data_ptr()), [hex(p) for p in h2.buffer_ptrs], hex(h2.multicast_ptr or 0), flush=True)
dist.barrier()
dist.destroy_process_group()
