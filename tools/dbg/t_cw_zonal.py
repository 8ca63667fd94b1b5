import sys, os, json, torch
sys.path.insert(0, os.getcwd())
import paper_1606_05562_b200 as pkg, synth
pkg.dct16a_set_option(pkg.OPT_CODEC_PATH, 2)
x = torch.from_numpy(synth.video_u8(100)).cuda()
for r in (32, 100):
    rec, sse, ps = pkg.codec(x, "zonal", r=r, valid_height=1080)
    q = pkg.make_quant("zonal", r); d = pkg.desc_of(x, valid_height=1080)
    s = torch.empty(100, dtype=torch.int64, device="cuda")
    for _ in range(3): pkg.dct16a_codec(x, q, s, rec, None, d)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10): pkg.dct16a_codec(x, q, s, rec, None, d)
    b.record(); b.synchronize()
    print(json.dumps({"r": r, "ms_100_frames_warp_kernel": a.elapsed_time(b) / 10}))
