import sys; sys.path.insert(0,'.')
import numpy as np, torch
import paper_1606_05562_b200 as pkg, synth
from oracle import codec as oc
imgs = synth.image_u8(0)[None]
x = torch.from_numpy(imgs).cuda()
for path in (0,3):
    pkg.dct16a_set_option(pkg.OPT_CODEC_PATH, path)
    rec, sse, ps = pkg.codec(x, "zonal", r=16)
    torch.cuda.synchronize()
    ref = oc.codec_images(imgs, "zonal", r=16)
    r = rec.cpu().numpy(); d = r.astype(int) - ref["recon_img"].astype(int)
    bad = np.argwhere(d != 0)
    print(path, "mismatches", len(bad), "sse", sse.cpu().tolist(), ref["sse"])
    if len(bad):
        print(bad[:10]); blk = bad[0]
        bi, bj = blk[1]//16, blk[2]//16
        print("block", bi, bj); print(d[0, bi*16:bi*16+16, bj*16:bj*16+16])
