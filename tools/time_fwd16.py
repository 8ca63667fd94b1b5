"""Config-2 throughput of dct16a_forward16 (16-bit coefficients: 768 B/block)
next to dct16a_forward (int32: 1280 B/block); CUDA events, 100 launches."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1606_05562_b200 as pkg  # noqa: E402
import synth  # noqa: E402

x = torch.from_numpy(synth.batch_u8(range(4096), 512, 512)).cuda()
nb = 4096 * 1024
d = pkg.desc_of(x)
for name, out, bpb, fn in [("forward16", torch.empty((nb, 16, 16), dtype=torch.int16, device="cuda"), 768,
                            pkg.dct16a_forward16),
                           ("forward", torch.empty((nb, 16, 16), dtype=torch.int32, device="cuda"), 1280,
                            pkg.dct16a_forward)]:
    for _ in range(5):
        fn(x, out, d)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(100):
        fn(x, out, d)
    b.record()
    b.synchronize()
    ms = a.elapsed_time(b) / 100
    print(json.dumps({"entry": name, "ms": ms, "blocks_per_s": nb / ms * 1e3, "alg_GBs": nb * bpb / ms / 1e6}))
    del out
