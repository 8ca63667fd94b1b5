import torch
x = torch.empty(4096*512*512, dtype=torch.int32, device="cuda")
def t(f, reps=20):
    f(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): f()
    b.record(); b.synchronize()
    return a.elapsed_time(b) / reps
n = x.numel() * 4
for name, f in [("fill_(7)", lambda: x.fill_(7)), ("zero_", lambda: x.zero_()),
                ("copy_(arange-ish)", None)]:
    if f is None: continue
    ms = t(f); print(name, ms, n / ms / 1e6, "GB/s")
y = torch.randint(0, 1 << 30, (x.numel(),), dtype=torch.int32, device="cuda")
ms = t(lambda: x.copy_(y)); print("copy random 4GiB", ms, 2 * n / ms / 1e6, "GB/s r+w")
z = torch.randint(0, 256, (x.numel(),), dtype=torch.uint8, device="cuda")
ms = t(lambda: x.copy_(z)); print("u8->i32 copy_", ms, 5 * x.numel() / ms / 1e6, "GB/s mix")
