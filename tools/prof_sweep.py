"""Profiling driver: config-5 r-sweep launches (dct16a_zonal_sweep, r = 1..256) on
16 of the 64 images, nothing else.  Used under ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1606_05562_b200 as pkg  # noqa: E402
import synth  # noqa: E402

x = torch.from_numpy(synth.batch_u8(range(100, 116), 1024, 1024, rho=synth.cfg5_rho)).cuda()
for _ in range(2):
    s, p = pkg.zonal_sweep(x, 1, 256)
torch.cuda.synchronize()
print("ok", int(s.sum()))
