"""Forward transform of 10-bit frames (200 x 3840x2160 int16, config-4 recipe)
under each K1 output path (DCT16A_OPT_FWD_STORE), CUDA events."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1606_05562_b200 as pkg  # noqa: E402
import synth  # noqa: E402

x = torch.from_numpy(synth.frames_10bit(range(200))).cuda()
nb = 200 * 135 * 240
coef = torch.empty((nb, 16, 16), dtype=torch.int32, device="cuda")
d = pkg.desc_of(x)
ref = None
for mode in (0, 1, 3, 4, 5, 7):
    pkg.dct16a_set_option(pkg.OPT_FWD_STORE, mode)
    for _ in range(3):
        pkg.dct16a_forward(x, coef, d)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        pkg.dct16a_forward(x, coef, d)
    b.record()
    b.synchronize()
    ms = a.elapsed_time(b) / 20
    chk = int(coef[::9973].to(torch.int64).sum())
    ref = chk if ref is None else ref
    print(json.dumps({"mode": mode, "ms": ms, "GBs": nb * 1536 / ms / 1e6, "same": chk == ref}), flush=True)
