"""Build kernel variants of libdct16a.so (extra -D macros) into build/variants/
and time one workload per variant in a fresh process each (DCT16A_LIB).
  python tools/variants.py build NAME=DEF1,DEF2 ...
  python tools/variants.py time --config 4 --frames 200
"""
import glob
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
VDIR = os.path.join(ROOT, "build", "variants")
sys.path.insert(0, ROOT)

TIMER = r"""
import sys, json, torch
sys.path.insert(0, %r)
import paper_1606_05562_b200 as pkg, synth
cfg, frames = %d, %d
if cfg == 2:
    x = torch.from_numpy(synth.batch_u8(range(4096), 512, 512)).cuda()
    coef = torch.empty((4096 * 1024, 16, 16), dtype=torch.int32, device="cuda")
    d = pkg.desc_of(x)
    for _ in range(5): pkg.dct16a_forward(x, coef, d)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(100): pkg.dct16a_forward(x, coef, d)
    b.record(); b.synchronize()
    ms = a.elapsed_time(b) / 100
    print(json.dumps({"ms": ms, "GBs": 4096 * 1024 * 1280 / ms / 1e6, "chk": int(coef[12345].sum()) + int(coef[-1].sum())}))
    sys.exit(0)
if cfg == 4:
    x = torch.from_numpy(synth.frames_10bit(range(frames))).cuda(); q = pkg.make_quant("uniform", step=16); vh = None
else:
    x = torch.from_numpy(synth.video_u8(frames)).cuda(); q = pkg.make_quant("zonal", %d); vh = 1080
n = x.shape[0]; rec = torch.empty_like(x)
sse = torch.empty(n, dtype=torch.int64, device="cuda"); ps = torch.empty(n, dtype=torch.float64, device="cuda")
d = pkg.desc_of(x, valid_height=vh)
for _ in range(3): pkg.dct16a_codec(x, q, sse, rec, ps, d)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10): pkg.dct16a_codec(x, q, sse, rec, ps, d)
b.record(); b.synchronize()
print(json.dumps({"ms": a.elapsed_time(b) / 10, "sse0": int(sse[0]), "sum": int(sse.sum())}))
"""


def main():
    if sys.argv[1] == "build":
        from paper_1606_05562_b200 import build as b
        os.makedirs(VDIR, exist_ok=True)
        for spec in sys.argv[2:]:
            name, _, defs = spec.partition("=")
            out = os.path.join(VDIR, f"lib_{name}.so")
            b.build(out=out, defines=[d for d in defs.split(",") if d])
            print("built", out)
    else:
        import argparse
        ap = argparse.ArgumentParser()
        ap.add_argument("cmd")
        ap.add_argument("--config", type=int, default=4)
        ap.add_argument("--frames", type=int, default=200)
        ap.add_argument("--r", type=int, default=32)
        a = ap.parse_args()
        libs = [("default", os.path.join(ROOT, "paper_1606_05562_b200", "libdct16a.so"))] + \
            [(os.path.basename(p)[4:-3], p) for p in sorted(glob.glob(os.path.join(VDIR, "lib_*.so")))]
        for name, lib in libs:
            env = dict(os.environ, DCT16A_LIB=lib)
            r = subprocess.run([sys.executable, "-c", TIMER % (ROOT, a.config, a.frames, a.r)], env=env,
                               capture_output=True, text=True)
            out = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr.strip()[-300:]
            print(json.dumps({"variant": name, "result": out}), flush=True)


if __name__ == "__main__":
    main()
