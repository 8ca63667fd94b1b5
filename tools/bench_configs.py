"""Per-config throughput of every hot-path entry on B200: the forward kernel
(config 2), the fused codec (configs 1, 3, 4) and the r-sweep (config 5),
device-resident inputs, CUDA events; beside each, the CPU oracle (as it
stands, numpy float64 / exact integers, one process per host core) on a
bounded sample of the same workload.  One JSON object per config.  Secondary
measurements: bench.py times config 2 under the driver contract."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
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


CORES = len(os.sched_getaffinity(0))


def oracle_items(c):
    return {1: 1, 2: 1024, 3: 32, 4: 16, 5: 16}[c]


def _oracle_job(args):
    from threadpoolctl import threadpool_limits

    from oracle import codec as oc
    c, img, kw, vh = args
    with threadpool_limits(1):
        if c == 2:
            oc.forward(oc.to_blocks(img.astype(np.int64)))
        elif c == 5:
            for r in range(1, 257):
                oc.codec_images(img, "zonal", r=r)
        else:
            oc.codec_images(img, kw["mode"], r=kw.get("r", 16), step=kw.get("step", 16),
                            bit_depth=10 if kw["mode"] == "uniform" else 8, valid_height=vh)
    n, h, w = img.shape
    return n * (h // 16) * (w // 16) * (256 if c == 5 else 1)


def oracle_rate(c, xs, kw, vh):
    """The oracle as it stands on a bounded sample (one image/frame per job,
    one process per host core); returns (units/s over wall time, description)."""
    from concurrent.futures import ProcessPoolExecutor
    jobs = [(c, xs[i:i + 1], kw, vh) for i in range(xs.shape[0])]
    with ProcessPoolExecutor(min(CORES, len(jobs))) as ex:
        list(ex.map(_oracle_job, [(c, xs[:1, :16, :16], kw, None)] * min(CORES, len(jobs))))   # warm the workers
        t0 = time.time()
        units = sum(ex.map(_oracle_job, jobs))
        wall = time.time() - t0
    what = {1: "config-1 image", 2: "1024 config-2 images", 3: "32 config-3 frames", 4: "16 config-4 frames",
            5: "16 config-5 images x 256 r"}[c]
    return units / wall, f"{what}, {min(CORES, len(jobs))} processes, {wall:.1f} s wall"


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
        xs = x[:oracle_items(c)].cpu().numpy()
        o_rate, o_sample = oracle_rate(c, xs, kw if c in (1, 3, 4) else None, vh if c in (1, 3, 4) else None)
        gpu_rate = (blocks * 256 if c == 5 else blocks) / ms * 1e3
        print(json.dumps({"config": c, "blocks": blocks, "ms": ms, "blocks_per_s": blocks / ms * 1e3,
                          "alg_GBs": alg / ms / 1e6, "frac_of_measured_hbm": alg / ms / 1e6 / peak,
                          "gen_s": round(gen_s, 1), **extra,
                          "oracle": {"rate": o_rate, "unit": "block-evaluations/s" if c == 5 else "blocks/s",
                                     "sample": o_sample, "cores": CORES},
                          "gpu_over_oracle": gpu_rate / o_rate}), flush=True)
        del x
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
