"""Per-config throughput of the fused codec path (configs 1, 3, 4) and the
forward kernel (config 2), device-resident inputs, CUDA events.  Prints one
JSON object per config.  Secondary measurements (bench.py times config 2)."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1606_05562_b200 as pkg  # noqa: E402
import synth  # noqa: E402


def timeit(fn, reps, warm=3):
    for _ in range(warm):
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
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,3,4,5")
    ap.add_argument("--cfg3-frames", type=int, default=600)
    ap.add_argument("--cfg4-frames", type=int, default=1000)
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    for c in [int(v) for v in args.configs.split(",")]:
        t0 = time.time()
        if c == 1:
            x = torch.from_numpy(synth.image_u8(0)[None]).cuda()
            kw = dict(mode="zonal", r=16)
            vh = None
        elif c == 2:
            x = torch.from_numpy(synth.batch_u8(range(4096), 512, 512)).cuda()
        elif c == 3:
            x = torch.from_numpy(synth.video_u8(args.cfg3_frames)).cuda()
            kw = dict(mode="zonal", r=32)
            vh = 1080
        elif c == 5:
            x = torch.from_numpy(synth.config5_images()).cuda()
        elif c == 4:
            n = args.cfg4_frames
            x = torch.empty((n, 2160, 3840), dtype=torch.int16, device="cuda")
            step = 50
            for s in range(0, n, step):
                x[s:s + step] = torch.from_numpy(synth.frames_10bit(range(s, min(n, s + step)))).cuda()
            kw = dict(mode="uniform", step=16)
            vh = None
        gen_s = time.time() - t0
        n, h, w = x.shape
        blocks = n * (h // 16) * (w // 16)
        extra = {}
        if c == 2:
            coef = torch.empty((blocks, 16, 16), dtype=torch.int32, device="cuda")
            ms = timeit(lambda: pkg.dct16a_forward(x, coef, pkg.desc_of(x)), args.reps)
            alg = blocks * 1280
        elif c == 5:
            sse = torch.empty((n, 256), dtype=torch.int64, device="cuda")
            ps = torch.empty((n, 256), dtype=torch.float64, device="cuda")
            d = pkg.desc_of(x)
            ms = timeit(lambda: pkg.dct16a_zonal_sweep(x, 1, 256, sse, ps, d), args.reps)
            alg = blocks * 256
            extra = {"block_evals": blocks * 256, "block_evals_per_s": blocks * 256 / ms * 1e3}
        else:
            recon = torch.empty_like(x)
            d = pkg.desc_of(x, valid_height=vh)
            q = pkg.make_quant(kw["mode"], kw.get("r", 16), kw.get("step", 16))
            sse = torch.empty(n, dtype=torch.int64, device="cuda")
            ps = torch.empty(n, dtype=torch.float64, device="cuda")
            ms = timeit(lambda: pkg.dct16a_codec(x, q, sse, recon, ps, d), args.reps)
            alg = blocks * 2 * 256 * x.element_size()
        print(json.dumps({"config": c, "blocks": blocks, "ms": ms, "blocks_per_s": blocks / ms * 1e3,
                          "alg_GBs": alg / ms / 1e6, "frac_of_measured_hbm": alg / ms / 1e6 / peak,
                          "gen_s": round(gen_s, 1), **extra}), flush=True)
        del x
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
