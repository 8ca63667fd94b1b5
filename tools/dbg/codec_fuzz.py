"""Fuzz of the fused codec on every kernel path: random geometries
(ragged widths, pitched/strided windows, valid_height < H, batches 1-3),
8/10-bit, zonal (random r) and uniform (random step), smooth and noise content,
against the oracle byte for byte."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1606_05562_b200 as pkg  # noqa: E402
from oracle import codec as oc  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 100
# the product library's kernel choices; an experiment build (DCT16A_LIB) adds 1, 3, 4
PATHS = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0, 2]
rng = np.random.default_rng(int(sys.argv[3]) if len(sys.argv) > 3 else 777)
MAXSTEP = int(sys.argv[4]) if len(sys.argv) > 4 else 119   # uniform steps drawn from [1, MAXSTEP]
bad = 0
for c in range(cases):
    bd = 8 if rng.random() < 0.5 else 10
    hi = 256 if bd == 8 else 1024
    dt = np.uint8 if bd == 8 else np.int16
    n = int(rng.integers(1, 4))
    H = 16 * int(rng.integers(1, 7))
    W = 16 * int(rng.integers(1, 30))
    pad = (16 if bd == 8 else 8) * int(rng.integers(0, 3))
    base = rng.integers(0, hi, size=(n, H + int(rng.integers(0, 3)), W + pad)).astype(dt)
    if rng.random() < 0.5:
        f = np.cumsum(np.cumsum(rng.normal(size=base.shape), axis=1), axis=2)
        base = np.rint((f - f.min()) / max(1e-9, np.ptp(f)) * (hi - 1)).astype(dt)
    view = np.ascontiguousarray(base[:, :H, :W])
    t = torch.from_numpy(base).cuda()[:, :H, :W]
    mode = "zonal" if rng.random() < 0.5 else "uniform"
    u = rng.random()
    r = int(rng.integers(1, 257)) if u < 0.3 else (int(rng.integers(1, 37)) if u < 0.6 else int(rng.integers(37, 137)))
    step = int(rng.integers(1, MAXSTEP + 1))
    vh = int(rng.integers(1, H + 1)) if rng.random() < 0.3 else None
    ref = oc.codec_images(view, mode, r=r, step=step, bit_depth=bd, valid_height=vh)
    for path in PATHS:
        pkg.dct16a_set_option(pkg.OPT_CODEC_PATH, path)
        rec, sse, _ = pkg.codec(t, mode, r=r, step=step, valid_height=vh)
        torch.cuda.synchronize()
        ok = np.array_equal(rec.cpu().numpy(), ref["recon_img"]) and sse.cpu().tolist() == ref["sse"]
        if not ok:
            bad += 1
            print("MISMATCH", c, path, bd, mode, n, H, W, r, step, vh)
pkg.dct16a_set_option(pkg.OPT_CODEC_PATH, 0)
print(f"codec fuzz: {cases} cases x {len(PATHS)} paths {PATHS}, {bad} mismatches")
