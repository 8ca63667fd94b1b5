import glob, os, subprocess, sys, json
T = r"""
import sys, torch
sys.path.insert(0, '.')
import paper_1606_05562_b200 as pkg, synth
x = torch.from_numpy(synth.config5_images()).cuda()
n = x.shape[0]
sse = torch.empty((n, 256), dtype=torch.int64, device='cuda'); ps = torch.empty((n, 256), dtype=torch.float64, device='cuda')
d = pkg.desc_of(x)
for _ in range(3): pkg.dct16a_zonal_sweep(x, 1, 256, sse, ps, d)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10): pkg.dct16a_zonal_sweep(x, 1, 256, sse, ps, d)
b.record(); b.synchronize()
print(a.elapsed_time(b) / 10, int(sse.sum()))
"""
libs = [("default", "paper_1606_05562_b200/libdct16a.so")] + [(os.path.basename(p), p) for p in sorted(glob.glob("build/variants/*.so"))]
for name, lib in libs:
    r = subprocess.run([sys.executable, "-c", T], env=dict(os.environ, DCT16A_LIB=os.path.abspath(lib)), capture_output=True, text=True)
    print(name, r.stdout.strip() or r.stderr[-300:])
