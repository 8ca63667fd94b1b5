import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import synth, paper_1606_05562_b200 as pkg
from oracle import codec as oc
pkg.dct16a_set_option(pkg.OPT_CODEC_PATH, 2)
cases = [("u8 r37", np.concatenate([synth.batch_u8([40, 41], 48, 272), synth.adversarial_u8(48, 272)]), "zonal", 8, 37, 16),
         ("u8 r37 w256", synth.batch_u8([40, 41], 48, 256), "zonal", 8, 37, 16),
         ("u8 r16 w128", synth.batch_u8([40], 16, 128), "zonal", 8, 16, 16),
         ("u8 r256 w128", synth.batch_u8([40], 16, 128), "zonal", 8, 256, 16),
         ("10b uni", synth.frames_10bit([6], H=64, W=128, workers=1), "uniform", 10, 16, 16)]
for name, imgs, mode, bd, r, step in cases:
    x = torch.from_numpy(imgs).cuda()
    rec, sse, ps = pkg.codec(x, mode, r=r, step=step)
    torch.cuda.synchronize()
    ref = oc.codec_images(imgs, mode, r=r, step=step, bit_depth=bd)
    g = rec.cpu().numpy().astype(np.int64); w = ref["recon_img"]
    bad = np.argwhere(g != w)
    print(name, "mismatches", len(bad), "sse", sse.cpu().tolist()[:3], ref["sse"][:3])
    if len(bad):
        n, i, j = bad[0]
        print("  first", bad[:5].tolist(), "images", sorted(set(bad[:, 0].tolist()))[:10],
              "rows", sorted(set((bad[:, 1] % 16).tolist())), "cols//16", sorted(set((bad[:, 2] // 16).tolist())))
        print("  got", g[n, i, max(0, j-4):j+4], "want", w[n, i, max(0, j-4):j+4], "orig", imgs[n, i, max(0, j-4):j+4])
