"""The staged ABI chain dct16a_forward -> dct16a_quantize -> dct16a_inverse ->
dct16a_psnr on config 3 (zonal r=32) and a 200-frame slice of config 4
(uniform, step 16): CUDA-event time of each entry and its algorithmic bytes
(int32 coefficients and levels through HBM), next to the fused dct16a_codec."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1606_05562_b200 as pkg  # noqa: E402
import synth  # noqa: E402


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


def main():
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    for name, x, q, vh in [
        ("config 3", torch.from_numpy(synth.video_u8(600)).cuda(), pkg.make_quant("zonal", 32), 1080),
        ("config 4 (200 frames)", torch.from_numpy(synth.frames_10bit(range(200))).cuda(),
         pkg.make_quant("uniform", step=16), None)]:
        n, h, w = x.shape
        nb = n * (h // 16) * (w // 16)
        px = x.element_size()
        d = pkg.desc_of(x, valid_height=vh)
        coef = torch.empty((nb, 16, 16), dtype=torch.int32, device="cuda")
        qc = torch.empty_like(coef)
        rec = torch.empty_like(x)
        sse = torch.empty(n, dtype=torch.int64, device="cuda")
        ps = torch.empty(n, dtype=torch.float64, device="cuda")
        steps = [("dct16a_forward", lambda: pkg.dct16a_forward(x, coef, d), nb * (256 * px + 1024)),
                 ("dct16a_quantize", lambda: pkg.dct16a_quantize(coef, qc, q, d), nb * 2048),
                 ("dct16a_inverse", lambda: pkg.dct16a_inverse(qc, rec, q, d), nb * (1024 + 256 * px)),
                 ("dct16a_psnr", lambda: pkg.dct16a_psnr(x, rec, sse, ps, d), nb * 512 * px),
                 ("dct16a_codec (fused)", lambda: pkg.dct16a_codec(x, q, sse, rec, ps, d), nb * 512 * px)]
        tot = 0.0
        for sname, fn, by in steps:
            ms = timeit(fn)
            if "fused" not in sname:
                tot += ms
            print(json.dumps({"case": name, "entry": sname, "ms": round(ms, 4), "alg_GBs": round(by / ms / 1e6, 1),
                              "frac_hbm": round(by / ms / 1e6 / peak, 3)}), flush=True)
        print(json.dumps({"case": name, "entry": "chain total", "ms": round(tot, 4)}), flush=True)
        del x, coef, qc, rec
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
