"""Small invocation of every entry point of libdct16a for compute-sanitizer
(one tool per run, e.g. `compute-sanitizer --tool memcheck python
tools/sanitize_run.py`): forward 8/10-bit with ragged tiles and pitched views,
quantize/inverse (zonal, uniform), psnr, the fused codec on all three kernel
choices, the r-sweep and SSIM.  Prints a checksum; parity is the tests' job."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1606_05562_b200 as pkg  # noqa: E402
import synth  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    u8 = torch.from_numpy(synth.batch_u8([1, 2], 48, 272, workers=1)).to(dev)
    f10 = torch.from_numpy(synth.frames_10bit([3], H=32, W=208, workers=1)).to(dev)
    big = torch.from_numpy(synth.batch_u8([4], 64, 400, workers=1)).to(dev)
    view = big[:, 8:56, 32:288]
    chk = 0
    for x, bd in ((u8, 8), (f10, 10), (view, 8)):
        coef = pkg.forward(x)
        chk += int(coef.sum())
        n, h, w = x.shape
        nb = coef.shape[0]
        d = pkg.desc_of(x, bd)
        for mode, r, step in (("zonal", 21, 16), ("uniform", 16, 16)):
            q = pkg.make_quant(mode, r, step)
            qc = torch.empty_like(coef)
            sc = torch.empty((nb, 16, 16), dtype=torch.float32, device=dev)
            rec = torch.empty((n, h, w), dtype=x.dtype, device=dev)
            pkg.dct16a_quantize(coef, qc, q, d, sc)
            pkg.dct16a_inverse(qc, rec, q, pkg.desc_of(rec, bd))
            sse = torch.empty(n, dtype=torch.int64, device=dev)
            ps = torch.empty(n, dtype=torch.float64, device=dev)
            pkg.dct16a_psnr(x.contiguous(), rec, sse, ps, pkg.desc_of(rec, bd))
            chk += int(sse.sum())
            for path in (0, 1, 2, 3):
                pkg.dct16a_set_option(pkg.OPT_CODEC_PATH, path)
                for r2 in (16, 40):
                    rec2, sse2, _ = pkg.codec(x.contiguous(), mode, r=r2, step=step)
                    chk += int(sse2.sum())
            pkg.dct16a_set_option(pkg.OPT_CODEC_PATH, 0)
        s, _ = pkg.zonal_sweep(x.contiguous(), 1, 40)
        chk += int(s.sum())
        chk += int(1e6 * float(pkg.ssim(x.contiguous(), rec).sum()))
    torch.cuda.synchronize()
    print("sanitize run ok, checksum", chk)


if __name__ == "__main__":
    main()
