"""Config-5 r-sweep timing (dct16a_zonal_sweep, r = 1..256) on B200: the 64
config-5 images (8-bit) and 16 10-bit 1024² frames, CUDA events per call, plus
a checksum of every SSE so that builds can be compared (parity against the
oracle lives in tests/test_gpu_parity.py).  One JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1606_05562_b200 as pkg  # noqa: E402
import synth  # noqa: E402


def timeit(fn, reps=10, warm=3):
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


x8 = torch.from_numpy(synth.config5_images()).cuda()
x10 = torch.from_numpy(synth.frames_10bit(range(16), H=1024, W=1024)).cuda()
out = {"lib": pkg._lib.LIB_PATH}
for name, x in (("cfg5_u8", x8), ("u16_16x1024", x10)):
    ms = timeit(lambda: pkg.zonal_sweep(x, 1, 256))
    s, _ = pkg.zonal_sweep(x, 1, 256)
    s2, _ = pkg.zonal_sweep(x, 37, 100)   # a range that is not a multiple of the unroll
    torch.cuda.synchronize()
    out[name] = {"ms": ms, "sse_sum": int(s.sum()), "sse_hash": int((s * torch.arange(1, 257, device="cuda")).sum() % (1 << 61)),
                 "sub_range_equal": bool(torch.equal(s2, s[:, 36:136]))}
print(json.dumps(out))
