"""Profiling driver: the staged chain (forward, quantize, inverse, psnr) on 100
config-3 frames (zonal r=32) or 50 config-4 frames (uniform), nothing else."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1606_05562_b200 as pkg  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
a = ap.parse_args()
if a.config == 3:
    x = torch.from_numpy(synth.video_u8(100)).cuda()
    q, vh = pkg.make_quant("zonal", 32), 1080
else:
    x = torch.from_numpy(synth.frames_10bit(range(50))).cuda()
    q, vh = pkg.make_quant("uniform", step=16), None
n, h, w = x.shape
nb = n * (h // 16) * (w // 16)
d = pkg.desc_of(x, valid_height=vh)
coef = torch.empty((nb, 16, 16), dtype=torch.int32, device="cuda")
qc = torch.empty_like(coef)
rec = torch.empty_like(x)
sse = torch.empty(n, dtype=torch.int64, device="cuda")
for _ in range(2):
    pkg.dct16a_forward(x, coef, d)
    pkg.dct16a_quantize(coef, qc, q, d)
    pkg.dct16a_inverse(qc, rec, q, d)
    pkg.dct16a_psnr(x, rec, sse, None, d)
torch.cuda.synchronize()
print("ok", int(sse.sum()))
