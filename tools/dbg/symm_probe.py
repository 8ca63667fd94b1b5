import os, torch, torch.distributed as dist
import torch.distributed._symmetric_memory as sm
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29555")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
t = sm.empty(8, dtype=torch.int64, device="cuda")
h = sm.rendezvous(t, group=dist.group.WORLD)
print("multicast_ptr", getattr(h, "multicast_ptr", None), "buffer_ptrs", getattr(h, "buffer_ptrs", None))
print("has_multicast_support", sm.has_multicast_support(torch.device("cuda").type, 0) if hasattr(sm, "has_multicast_support") else "n/a")
dist.destroy_process_group()
