#!/usr/bin/env python
"""Config-4 fused uniform codec: the two-blocks-per-lane kernel (codec path 0,
codec_uniform.cu) against the warp-per-block-pair kernel (path 2,
codec_warp.cu) on F frames (fixture f mod D, D distinct AR(1) 10-bit frames),
CUDA events; every recon byte and SSE compared between the two paths, and
two frames against the oracle.  Also 8-bit uniform (config-2 images)."""
import argparse
import json
import os
import sys

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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=300)
    ap.add_argument("--distinct", type=int, default=16)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--oracle", type=int, default=1)
    ap.add_argument("--steps", default="16")
    ap.add_argument("--paths", default="0,2", help="two codec paths to compare (4 = experiment build)")
    a = ap.parse_args()
    d = torch.from_numpy(synth.frames_10bit(range(a.distinct))).cuda()
    x = d[torch.arange(a.frames, device="cuda") % a.distinct]
    res = {"frames": a.frames}
    for step in [int(v) for v in a.steps.split(",")]:
        q = pkg.make_quant("uniform", step=step)
        out = {}
        P0, P1 = [int(v) for v in a.paths.split(",")]
        for path in (P0, P1):
            pkg.dct16a_set_option(pkg.OPT_CODEC_PATH, path)
            rec = torch.empty_like(x)
            sse = torch.empty(a.frames, dtype=torch.int64, device="cuda")
            ms = timeit(lambda: pkg.dct16a_codec(x, q, sse, rec, None, pkg.desc_of(x)), a.reps)
            out[path] = (ms, rec, sse)
        pkg.dct16a_set_option(pkg.OPT_CODEC_PATH, 0)
        same = bool(torch.equal(out[P0][1], out[P1][1])) and bool(torch.equal(out[P0][2], out[P1][2]))
        r = {"ms_new": out[P0][0], "ms_old": out[P1][0], "paths_equal": same,
             "ms_per_1000_frames_new": out[P0][0] * 1000 / a.frames,
             "hbm_frac_new": a.frames * 32400 * 1024 / (out[P0][0] / 1e3) / 6548.2e9}
        if not same:
            diff = (out[P0][1] != out[P1][1]).nonzero()
            r["n_recon_diff"] = int(diff.shape[0])
            r["first_diff"] = diff[:5].tolist()
            r["sse_diff_frames"] = (out[P0][2] != out[P1][2]).nonzero().flatten()[:10].tolist()
        if a.oracle and step == 16:
            from oracle import codec as oc
            f = d[:a.oracle].cpu().numpy()
            ref = oc.codec_images(f, "uniform", step=16, bit_depth=10)
            r["oracle_recon_equal"] = bool(np.array_equal(out[P0][1][:a.oracle].cpu().numpy(), ref["recon_img"]))
            r["oracle_sse_equal"] = out[P0][2][:a.oracle].cpu().tolist() == ref["sse"]
        res[f"step{step}"] = r
    # 8-bit uniform on config-2 images
    x8 = torch.from_numpy(synth.batch_u8(range(256), 512, 512)).cuda()
    q = pkg.make_quant("uniform", step=16)
    o8 = {}
    P0, P1 = [int(v) for v in a.paths.split(",")]
    for path in (P0, P1):
        pkg.dct16a_set_option(pkg.OPT_CODEC_PATH, path)
        rec = torch.empty_like(x8)
        sse = torch.empty(256, dtype=torch.int64, device="cuda")
        o8[path] = (timeit(lambda: pkg.dct16a_codec(x8, q, sse, rec, None, pkg.desc_of(x8)), a.reps), rec, sse)
    pkg.dct16a_set_option(pkg.OPT_CODEC_PATH, 0)
    res["u8_256img"] = {"ms_new": o8[P0][0], "ms_old": o8[P1][0],
                        "paths_equal": bool(torch.equal(o8[P0][1], o8[P1][1])) and bool(torch.equal(o8[P0][2], o8[P1][2]))}
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
