"""Profiling driver: N fused-codec launches on config 3 (zonal r=32) or
config 4 (uniform, --frames frames), or N r-sweeps on config 5 (--config 5:
--frames images of 1024x1024, r = 1..256), nothing else.  Used under ncu."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1606_05562_b200 as pkg  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--frames", type=int, default=100)
ap.add_argument("--launches", type=int, default=2)
ap.add_argument("--step", type=int, default=16, help="config 4: uniform step")
args = ap.parse_args()
if args.config == 5:
    x = torch.from_numpy(synth.config5_images()[:args.frames]).cuda()
    for _ in range(args.launches):
        pkg.zonal_sweep(x, 1, 256)
    torch.cuda.synchronize()
    print("ok sweep")
    sys.exit(0)
if args.config == 3:
    x = torch.from_numpy(synth.video_u8(args.frames)).cuda()
    q, vh = pkg.make_quant("zonal", 32), 1080
else:
    x = torch.from_numpy(synth.frames_10bit(range(args.frames))).cuda()
    q, vh = pkg.make_quant("uniform", step=args.step), None
n = x.shape[0]
recon = torch.empty_like(x)
sse = torch.empty(n, dtype=torch.int64, device="cuda")
ps = torch.empty(n, dtype=torch.float64, device="cuda")
d = pkg.desc_of(x, valid_height=vh)
for _ in range(args.launches):
    pkg.dct16a_codec(x, q, sse, recon, ps, d)
torch.cuda.synchronize()
print("ok", float(ps[0]))
