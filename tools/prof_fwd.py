"""Profiling driver: N launches of the config-2 forward kernel (and, with
--codec, one fused codec launch per config), nothing else.  Used under ncu."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1606_05562_b200 as pkg  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--launches", type=int, default=3)
ap.add_argument("--images", type=int, default=4096)
args = ap.parse_args()
x = torch.from_numpy(synth.batch_u8(range(args.images), 512, 512)).cuda()
coef = torch.empty((args.images * 1024, 16, 16), dtype=torch.int32, device="cuda")
for _ in range(args.launches):
    pkg.dct16a_forward(x, coef, pkg.desc_of(x))
torch.cuda.synchronize()
print("ok", int(coef[0, 0, 0]))
