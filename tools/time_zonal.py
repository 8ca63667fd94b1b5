"""Zonal fused-codec kernels side by side (DCT16A_OPT_CODEC_PATH 0/2/3) on
configs 1 and 3: CUDA-event time per launch, device-resident input, and a
byte-for-byte cross-check of the reconstructions and SSE vectors between the
paths (the oracle parity lives in tests/test_gpu_parity.py).  One JSON line per
(config, path)."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1606_05562_b200 as pkg  # noqa: E402
import synth  # noqa: E402

NAMES = {0: "band (auto)", 1: "generic", 2: "warp", 3: "tpb"}


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
    ap.add_argument("--frames", type=int, default=600)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--paths", default="0,2")
    ap.add_argument("--r", default="16,32,64,128")
    ap.add_argument("--bits", type=int, default=8, help="10: config-3 geometry with 10-bit frames (config-4 recipe)")
    args = ap.parse_args()
    peak = 6548.2
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        peak = json.load(open(p)).get("hbm_gbs", peak)
    if args.bits == 8:
        cases = [("config 1", torch.from_numpy(synth.image_u8(0)[None]).cuda(), None),
                 ("config 3", torch.from_numpy(synth.video_u8(args.frames)).cuda(), 1080)]
    else:
        f = torch.from_numpy(synth.frames_10bit(range(16), H=1088, W=1920)).cuda()
        cases = [("10-bit 1088x1920", f[torch.arange(args.frames, device="cuda") % 16], None)]
    old = pkg.dct16a_get_option(pkg.OPT_CODEC_PATH)
    for name, x, vh in cases:
        n, h, w = x.shape
        blocks = n * (h // 16) * (w // 16)
        d = pkg.desc_of(x, valid_height=vh)
        for r in [int(v) for v in args.r.split(",")]:
            q = pkg.make_quant("zonal", r, 16)
            ref = None
            for path in [int(v) for v in args.paths.split(",")]:
                pkg.dct16a_set_option(pkg.OPT_CODEC_PATH, path)
                recon = torch.empty_like(x)
                sse = torch.empty(n, dtype=torch.int64, device="cuda")
                ps = torch.empty(n, dtype=torch.float64, device="cuda")
                ms = timeit(lambda: pkg.dct16a_codec(x, q, sse, recon, ps, d), args.reps)
                same = None
                if ref is None:
                    ref = (recon.clone(), sse.clone())
                else:
                    same = bool(torch.equal(recon, ref[0]) and torch.equal(sse, ref[1]))
                gbs = blocks * 512 / ms / 1e6
                print(json.dumps({"case": name, "r": r, "path": path, "kernel": NAMES[path], "ms": ms,
                                  "blocks_per_s": blocks / ms * 1e3, "alg_GBs": gbs, "frac_hbm": gbs / peak,
                                  "matches_first_path": same}), flush=True)
    pkg.dct16a_set_option(pkg.OPT_CODEC_PATH, old)


if __name__ == "__main__":
    main()
