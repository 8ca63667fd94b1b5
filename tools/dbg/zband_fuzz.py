"""Fuzz of the band-pruned zonal kernel (codec path 0, 8- and 10-bit, every r):
random geometries (ragged widths, pitched/strided windows, valid_height < H,
batches 1-4, smooth and noise content) against the oracle, byte for byte."""
import sys

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1606_05562_b200 as pkg  # noqa: E402
from oracle import codec as oc  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 4242)
bad = 0
for c in range(cases):
    bd = 8 if rng.random() < 0.5 else 10
    hi, dt = (256, np.uint8) if bd == 8 else (1024, np.int16)
    n = int(rng.integers(1, 5))
    H = 16 * int(rng.integers(1, 9))
    W = 16 * int(rng.integers(1, 40))
    pad = (16 if bd == 8 else 8) * int(rng.integers(0, 3))
    base = rng.integers(0, hi, size=(n, H + int(rng.integers(0, 3)), W + pad)).astype(dt)
    if rng.random() < 0.5:
        f = np.cumsum(np.cumsum(rng.normal(size=base.shape), axis=1), axis=2)
        base = np.rint((f - f.min()) / max(1e-9, np.ptp(f)) * (hi - 1)).astype(dt)
    view = np.ascontiguousarray(base[:, :H, :W])
    t = torch.from_numpy(base).cuda()[:, :H, :W]
    r = int(rng.integers(1, 257))
    vh = int(rng.integers(1, H + 1)) if rng.random() < 0.3 else None
    rec, sse, _ = pkg.codec(t, "zonal", r=r, valid_height=vh)
    torch.cuda.synchronize()
    ref = oc.codec_images(view, "zonal", r=r, valid_height=vh, bit_depth=bd)
    ok = np.array_equal(rec.cpu().numpy(), ref["recon_img"]) and sse.cpu().tolist() == ref["sse"]
    if not ok:
        bad += 1
        print("MISMATCH", c, n, H, W, r, vh)
print(f"zband fuzz: {cases} cases, {bad} mismatches")
