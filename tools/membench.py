"""Memory-roofline microbenchmarks for the config-2 byte mix (1 GiB read,
4 GiB write): what simple torch kernels reach on this GPU."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def timeit(fn, reps=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


res = {}
n = 1 << 30
x8 = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda")
y32 = torch.empty(n, dtype=torch.int32, device="cuda")
bf = torch.randn(n, dtype=torch.bfloat16, device="cuda")
bf2 = torch.empty_like(bf)
ms = timeit(lambda: bf2.copy_(bf))
res["copy_bf16_1Gi_GBs"] = 4 * n / ms / 1e6
ms = timeit(lambda: y32.copy_(x8))
res["u8_to_i32_1Gi_GBs(5GB mix)"] = 5 * n / ms / 1e6
ms = timeit(lambda: y32.fill_(7))
res["fill_i32_4GiB_GBs"] = 4 * n / ms / 1e6
ms = timeit(lambda: x8.sum(dtype=torch.int64))
res["read_u8_1GiB_GBs"] = n / ms / 1e6
print(json.dumps(res, indent=1))
