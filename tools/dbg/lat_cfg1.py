"""Config-1 latency (one 512x512 u8 image, fused zonal r = 16): where the
per-call time goes.  Prints: the Python codec() call, the C-ABI call with
preallocated outputs (wall per call, back to back), one call synchronised
each time, and a CUDA-graph replay of the C-ABI call (device time per replay)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1606_05562_b200 as pkg  # noqa: E402
from paper_1606_05562_b200 import _lib  # noqa: E402
import synth  # noqa: E402


def wall(fn, n):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / n * 1e6


def main():
    x = torch.from_numpy(synth.image_u8(0)[None]).cuda()
    d = pkg.desc_of(x)
    q = pkg.make_quant("zonal", 16, 16)
    sse = torch.empty(1, dtype=torch.int64, device="cuda")
    psnr = torch.empty(1, dtype=torch.float64, device="cuda")
    rec = torch.empty_like(x)
    out = {}
    out["python_codec_us"] = wall(lambda: pkg.codec(x, "zonal", r=16), 2000)
    out["cabi_call_us"] = wall(lambda: _lib.dct16a_codec(x, q, sse, rec, psnr, d), 2000)
    lib = _lib.lib()
    import ctypes
    args = (ctypes.c_void_p(x.data_ptr()), ctypes.byref(d), ctypes.byref(q), ctypes.c_void_p(rec.data_ptr()),
            ctypes.c_void_p(sse.data_ptr()), ctypes.c_void_p(psnr.data_ptr()), ctypes.c_void_p(0))
    out["raw_ctypes_us"] = wall(lambda: lib.dct16a_codec(*args), 2000)

    def one_sync():
        lib.dct16a_codec(*args)
        torch.cuda.synchronize()
    out["call_plus_sync_us"] = wall(one_sync, 500)
    # graph replay (static schedule), device time per replay
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        g = torch.cuda.CUDAGraph()
        _lib.dct16a_codec(x, q, sse, rec, psnr, d, s)   # warm
        s.synchronize()
        with torch.cuda.graph(g, stream=s):
            _lib.dct16a_codec(x, q, sse, rec, psnr, d, s)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(20):
        g.replay()
    torch.cuda.synchronize()
    a.record()
    for _ in range(1000):
        g.replay()
    b.record()
    b.synchronize()
    out["graph_replay_us"] = a.elapsed_time(b) / 1000 * 1e3
    ref = pkg.codec(x, "zonal", r=16)
    torch.cuda.synchronize()
    out["graph_result_ok"] = bool(torch.equal(rec, ref[0]) and int(sse[0]) == int(ref[1][0]))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
