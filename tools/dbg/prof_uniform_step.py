import sys; sys.path.insert(0, '.')
import torch, synth, paper_1606_05562_b200 as pkg
x = torch.from_numpy(synth.frames_10bit(range(8))).cuda()
q = pkg.make_quant("uniform", step=int(sys.argv[1]))
rec = torch.empty_like(x); sse = torch.empty(8, dtype=torch.int64, device="cuda")
for _ in range(2): pkg.dct16a_codec(x, q, sse, rec, None, pkg.desc_of(x))
torch.cuda.synchronize(); print("ok")
