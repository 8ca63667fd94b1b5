import torch, time
n = 4096 * 1024 * 256
dev = torch.device("cuda")
hd = torch.empty(n, dtype=torch.int32, pin_memory=True)
dd = torch.empty(n, dtype=torch.int32, device=dev)
hi = torch.empty(4096 * 512 * 512, dtype=torch.uint8, pin_memory=True)
di = torch.empty_like(hi, device=dev)
def t(f, reps=3):
    f(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): f()
    b.record(); b.synchronize()
    return a.elapsed_time(b) / reps
ms = t(lambda: hd.copy_(dd, non_blocking=True)); print("D2H 4GiB", ms, 4 * n / ms / 1e6, "GB/s")
ms = t(lambda: di.copy_(hi, non_blocking=True)); print("H2D 1GiB", ms, hi.numel() / ms / 1e6, "GB/s")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def both():
    with torch.cuda.stream(s1): hd.copy_(dd, non_blocking=True)
    with torch.cuda.stream(s2): di.copy_(hi, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
ms = t(both); print("D2H 4GiB || H2D 1GiB", ms, (4 * n + hi.numel()) / ms / 1e6, "GB/s total")
