"""Probe: torch symmetric memory + NVLS multicast on this box (world size 1)."""
import os
import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm_mem

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
torch.cuda.set_device(0)
from torch._C._distributed_c10d import _SymmetricMemory
print("has_multicast_support", _SymmetricMemory.has_multicast_support(torch._C._autograd.DeviceType.CUDA, 0))
print("backend", symm_mem.get_backend(torch.device("cuda:0")) if hasattr(symm_mem, "get_backend") else None)
t = symm_mem.empty(1024, dtype=torch.float32, device="cuda")
h = symm_mem.rendezvous(t, dist.group.WORLD.group_name)
print("rank", h.rank, "world", h.world_size)
print("multicast_ptr", hex(h.multicast_ptr) if h.multicast_ptr else h.multicast_ptr)
print("buffer_ptrs", [hex(x) for x in h.buffer_ptrs])
print("signal_pad_ptrs", [hex(x) for x in h.signal_pad_ptrs], "signal pad size", symm_mem.get_signal_pad_size())
print("attrs", [a for a in dir(h) if not a.startswith("_")])
dist.destroy_process_group()
