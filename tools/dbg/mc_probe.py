"""Probe: does this box expose CUDA multicast (NVLS) to a single process/GPU,
and does torch symmetric memory give a multicast address at world size 1?"""
import os
import torch
import torch.distributed as dist

from cuda.bindings import driver as cu

cu.cuInit(0)
err, dev = cu.cuDeviceGet(0)
err, mc = cu.cuDeviceGetAttribute(cu.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev)
print("cuInit/multicast supported:", err, mc)
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
import torch.distributed._symmetric_memory as symm
for backend in (None, "NVSHMEM", "CUDA"):
    try:
        if backend:
            symm.set_backend(backend)
        buf = symm.empty(1024, dtype=torch.int64, device="cuda")
        h = symm.rendezvous(buf, dist.group.WORLD)
        print("backend", backend, "multicast_ptr", getattr(h, "multicast_ptr", None), "peers", list(h.buffer_ptrs))
    except Exception as e:
        print("backend", backend, "error", type(e).__name__, str(e)[:200])
dist.destroy_process_group()
