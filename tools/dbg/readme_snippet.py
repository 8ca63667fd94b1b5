import sys; sys.path.insert(0, '.')
import torch, paper_1606_05562_b200 as dct16a

x = torch.randint(0, 256, (8, 1088, 1920), dtype=torch.uint8, device="cuda")
x10 = torch.randint(0, 1024, (4, 2160, 3840), dtype=torch.int16, device="cuda")
Z = dct16a.forward(x)                                   # int32 (8·68·120, 16, 16), Z = T·X·Tᵀ per block
Z16 = dct16a.forward16(x)                               # the same in 16 bits (DC as uint16)
rec, sse, psnr = dct16a.codec(x, "zonal", r=32, valid_height=1080)     # fused codec, exact pixels
ssim = dct16a.ssim(x, rec)                              # float64 per image
rec10, sse10, psnr10 = dct16a.codec(x10, "uniform", step=16)           # int16 10-bit frames
sse_r, psnr_r = dct16a.zonal_sweep(x, 1, 256)           # every r in one pass: (8, 256)
dct16a.dct16a_set_option(dct16a.OPT_UNIFORM_QUANT, 2)  # kernel choices never change results

torch.cuda.synchronize(); print('readme ok', float(psnr[0]), float(psnr10[0]), tuple(sse_r.shape), float(ssim[0]))
