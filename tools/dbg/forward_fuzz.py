"""Fuzz of the forward transform (dct16a_forward on both store paths, and the
16-bit dct16a_forward16 for 8-bit input) and of the r-sweep and SSIM on random
geometries (ragged widths up to 70 blocks, pitched/strided windows, batches
1-4, smooth / noise / saturated content) against the oracle, byte for byte
(SSIM within 1e-9).  usage: forward_fuzz.py N SEED"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1606_05562_b200 as pkg  # noqa: E402
from oracle import codec as oc  # noqa: E402
from oracle import quality as oq  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 9090)
bad = 0
for c in range(cases):
    bd = 8 if rng.random() < 0.5 else 10
    hi, dt = (256, np.uint8) if bd == 8 else (1024, np.int16)
    n = int(rng.integers(1, 5))
    H = 16 * int(rng.integers(1, 7))
    W = 16 * int(rng.integers(1, 71))
    pad = (16 if bd == 8 else 8) * int(rng.integers(0, 3))
    base = rng.integers(0, hi, size=(n, H + int(rng.integers(0, 3)), W + pad)).astype(dt)
    u = rng.random()
    if u < 0.4:
        f = np.cumsum(np.cumsum(rng.normal(size=base.shape), axis=1), axis=2)
        base = np.rint((f - f.min()) / max(1e-9, np.ptp(f)) * (hi - 1)).astype(dt)
    elif u < 0.5:
        base = np.where(rng.random(base.shape) < 0.5, 0, hi - 1).astype(dt)   # saturated
    view = np.ascontiguousarray(base[:, :H, :W])
    t = torch.from_numpy(base).cuda()[:, :H, :W]
    Z = oc.forward(oc.to_blocks(view.astype(np.int64))).reshape(-1, 16, 16)
    ok = True
    for store in (-1, 3, 5):
        pkg.dct16a_set_option(pkg.OPT_FWD_STORE, store)
        got = pkg.forward(t)
        torch.cuda.synchronize()
        ok &= np.array_equal(got.cpu().numpy(), Z)
    pkg.dct16a_set_option(pkg.OPT_FWD_STORE, -1)
    if bd == 8:
        g16 = pkg.forward16(t).cpu().numpy()
        dc = g16.view(np.uint16)[:, 0, 0].astype(np.int64)
        ac = g16.astype(np.int64)
        ac[:, 0, 0] = dc
        ok &= np.array_equal(ac, Z)
    if c % 10 == 0:   # the heavier checks on a sample
        r0, rc = int(rng.integers(1, 200)), int(rng.integers(1, 57))
        s, _ = pkg.zonal_sweep(t, r0, rc)
        ref = np.stack([oc.codec_images(view, "zonal", r=r, bit_depth=bd)["sse"] for r in range(r0, r0 + rc)], axis=1)
        ok &= np.array_equal(s.cpu().numpy(), ref)
        rec, _, _ = pkg.codec(t, "zonal", r=r0)
        ss = pkg.ssim(t, rec).cpu().numpy()
        ok &= bool(np.all(np.abs(ss - oq.ssim(view, rec.cpu().numpy(), bit_depth=bd)) < 1e-9))
    if not ok:
        bad += 1
        print("MISMATCH", c, bd, n, H, W, pad)
print(f"forward fuzz: {cases} cases (forward x 3 store paths, forward16, sweep and SSIM on every 10th), {bad} mismatches")
