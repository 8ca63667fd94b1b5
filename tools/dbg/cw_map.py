import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import synth, paper_1606_05562_b200 as pkg
from oracle import codec as oc
pkg.dct16a_set_option(pkg.OPT_CODEC_PATH, 2)
for (n, H, W, mode, r, bd) in [(1, 48, 272, "zonal", 37, 8), (1, 48, 272, "zonal", 16, 8), (1, 64, 144, "zonal", 16, 8),
                                (3, 48, 272, "zonal", 16, 8), (1, 48, 208, "uniform", 16, 10), (1, 64, 144, "uniform", 16, 8)]:
    imgs = synth.batch_u8(range(40, 40 + n), H, W) if bd == 8 else synth.frames_10bit(range(40, 40 + n), H=H, W=W, workers=1)
    x = torch.from_numpy(imgs).cuda()
    rec = torch.full_like(x, 7)
    sse = torch.empty(n, dtype=torch.int64, device="cuda"); ps = torch.empty(n, dtype=torch.float64, device="cuda")
    pkg.dct16a_codec(x, pkg.make_quant(mode, r, 16), sse, rec, ps, pkg.desc_of(x, bd))
    torch.cuda.synchronize()
    ref = oc.codec_images(imgs, mode, r=r, step=16, bit_depth=bd)
    g = rec.cpu().numpy().astype(np.int64); w = ref["recon_img"]
    bad = (g != w).reshape(n, H // 16, 16, W // 16, 16).any(axis=(2, 4))
    seven = (g == 7).reshape(n, H // 16, 16, W // 16, 16).all(axis=(2, 4))
    origm = (g == imgs).reshape(n, H // 16, 16, W // 16, 16).all(axis=(2, 4))
    print((n, H, W, mode, r, bd), "bad blocks", int(bad.sum()), "untouched(7)", int(seven.sum()), "==orig", int(origm.sum()))
    for img in range(n):
        for sy in range(H // 16):
            print("   ", img, sy, "".join("X" if bad[img, sy, b] else "." for b in range(W // 16)),
                  "".join("7" if seven[img, sy, b] else "." for b in range(W // 16)))
