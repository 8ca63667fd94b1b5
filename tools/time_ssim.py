"""Throughput of dct16a_ssim on the config-5 images (64 x 1024²) against their
r = 16 reconstructions, and on 100 config-3 frames; CUDA events."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1606_05562_b200 as pkg  # noqa: E402
import synth  # noqa: E402

for name, x, vh in [("config5 64x1024^2", torch.from_numpy(synth.config5_images()).cuda(), None),
                    ("config3 100x1920x1088", torch.from_numpy(synth.video_u8(100)).cuda(), 1080)]:
    rec, _, _ = pkg.codec(x, "zonal", r=16, valid_height=vh)
    out = torch.empty(x.shape[0], dtype=torch.float64, device="cuda")
    d = pkg.desc_of(x, valid_height=vh)
    for _ in range(3):
        pkg.dct16a_ssim(x, rec, out, d)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        pkg.dct16a_ssim(x, rec, out, d)
    b.record()
    b.synchronize()
    ms = a.elapsed_time(b) / 10
    n, h, w = x.shape
    win = n * ((vh or h) - 10) * (w - 10)
    print(json.dumps({"workload": name, "ms": ms, "windows_per_s": win / ms * 1e3, "mean_ssim": float(out.mean())}))
