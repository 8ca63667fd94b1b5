"""Times the forward kernel's output-path variants (store modes 0..7, set
through the DCT16A_FWD_STORE environment variable that initialises the
DCT16A_OPT_FWD_STORE option) on config-2-sized random images and prints a
result hash per mode (all equal).  One subprocess per mode."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import os, sys, json, torch
sys.path.insert(0, %r)
import paper_1606_05562_b200 as pkg
torch.manual_seed(0)
x = torch.randint(0, 256, (4096, 512, 512), dtype=torch.uint8, device="cuda")
coef = torch.empty((4096 * 1024, 16, 16), dtype=torch.int32, device="cuda")
d = pkg.desc_of(x)
for _ in range(5):
    pkg.dct16a_forward(x, coef, d)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(100):
    pkg.dct16a_forward(x, coef, d)
b.record(); b.synchronize()
ms = a.elapsed_time(b) / 100
h = int((coef.view(-1)[::9973].to(torch.int64) * torch.arange(coef.numel() // 9973 + 1, device="cuda")[: coef.view(-1)[::9973].numel()]).sum())
print(json.dumps({"ms": ms, "GBs": 4096 * 1024 * 1280 / ms / 1e6, "hash": h}))
"""

res = {}
for mode in sys.argv[1:] or [str(m) for m in range(8)]:
    env = dict(os.environ, DCT16A_FWD_STORE=mode)
    out = subprocess.run([sys.executable, "-c", CHILD % ROOT], env=env, capture_output=True, text=True)
    line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-500:]
    res[mode] = json.loads(line) if line.startswith("{") else line
print(json.dumps(res, indent=1))
