"""Probe: does torch symmetric memory give a multicast (NVLS) address on this
box, at world size 1 (one GPU per gpurun call)?  Prints the handle's fields."""
import os

import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm_mem

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
print("multicast attr:", torch.cuda.get_device_properties(dev))
for backend in (None, "CUDA", "NVSHMEM"):
    try:
        if backend:
            symm_mem.set_backend(backend)
        t = symm_mem.empty(1 << 16, dtype=torch.float64, device=dev)
        h = symm_mem.rendezvous(t, dist.group.WORLD.group_name)
        print(backend, "rank", h.rank, "world", h.world_size, "mc", hex(h.multicast_ptr), "bufs",
              [hex(p) for p in h.buffer_ptrs], "signal", [hex(p) for p in h.signal_pad_ptrs],
              "signal_pad_size", h.signal_pad_size)
    except Exception as e:  # noqa: BLE001
        print(backend, "error:", type(e).__name__, str(e)[:300])
dist.destroy_process_group()
