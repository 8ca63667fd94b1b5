"""paper_1606_05562_b200 — B200-native batched 16x16 approximate DCT of
arXiv 1606.05562 (multiplierless 16-point DCT approximation T, 60 additions).

The compute lives in libdct16a.so (hand-written sm_100a CUDA behind the C ABI
of include/dct16a.h); this package is the thin Python binding (``_lib``, same
names as the C entry points) plus allocation helpers.  PyTorch provides device
memory, streams and process groups only.
"""
from __future__ import annotations

from ._lib import (OPT_CODEC_PATH, OPT_FWD_STORE, OPT_UNIFORM_QUANT, UNIFORM, ZONAL, Dct16aError, Desc, Quant,  # noqa: F401
                   dct16a_codec, dct16a_codec_allreduce, dct16a_forward, dct16a_forward16, dct16a_forward_host,
                   dct16a_forward_host_workspace, dct16a_get_option, dct16a_inverse, dct16a_last_error, dct16a_psnr,
                   dct16a_quantize, dct16a_set_option, dct16a_sse_psnr, dct16a_ssim, dct16a_version, dct16a_zonal_sweep,
                   desc_of, lib, make_desc, make_quant)

__version__ = "0.2.0"


def forward(images, out=None, stream=None):
    """Z = T·X·Tᵀ for every 16x16 block of a (batch, H, W) uint8/int16 CUDA
    tensor; returns int32 (batch·H/16·W/16, 16, 16) block-major coefficients."""
    import torch
    if images.dim() == 2:
        images = images.unsqueeze(0)
    n, h, w = images.shape
    if out is None:
        out = torch.empty((n * (h // 16) * (w // 16), 16, 16), dtype=torch.int32, device=images.device)
    dct16a_forward(images, out, desc_of(images), stream)
    return out


def forward16(images, out=None, stream=None):
    """Z = T·X·Tᵀ of 8-bit images stored in 16 bits: int16 (batch·H/16·W/16,
    16, 16) block-major; entry [:, 0, 0] is the block sum as uint16 bits
    (use `.view(torch.uint16)` or `& 0xFFFF` on it), every other entry is int16."""
    import torch
    if images.dim() == 2:
        images = images.unsqueeze(0)
    n, h, w = images.shape
    if out is None:
        out = torch.empty((n * (h // 16) * (w // 16), 16, 16), dtype=torch.int16, device=images.device)
    dct16a_forward16(images, out, desc_of(images), stream)
    return out


def codec(images, mode="zonal", r=16, step=16, valid_height=None, want_recon=True, stream=None):
    """Fused forward -> quantise (S folded) -> inverse -> reconstruct -> SSE/PSNR.
    Returns (recon or None, sse int64[batch], psnr float64[batch])."""
    import torch
    if images.dim() == 2:
        images = images.unsqueeze(0)
    d = desc_of(images, valid_height=valid_height)
    n = images.shape[0]
    sse = torch.empty(n, dtype=torch.int64, device=images.device)
    psnr = torch.empty(n, dtype=torch.float64, device=images.device)
    # the C ABI describes src and recon with one descriptor: same strides
    recon = (torch.empty_strided(images.shape, images.stride(), dtype=images.dtype, device=images.device)
             if want_recon else None)
    dct16a_codec(images, make_quant(mode, r, step), sse, recon, psnr, d, stream)
    return recon, sse, psnr


def ssim(ref, test, bit_depth=None, valid_height=None, stream=None):
    """Mean SSIM per image of two (batch, H, W) CUDA tensors; float64 [batch]."""
    import torch
    if ref.dim() == 2:
        ref, test = ref.unsqueeze(0), test.unsqueeze(0)
    out = torch.empty(ref.shape[0], dtype=torch.float64, device=ref.device)
    dct16a_ssim(ref, test, out, desc_of(ref, bit_depth, valid_height), stream)
    return out


def zonal_sweep(images, r_first=1, r_count=256, valid_height=None, stream=None):
    """SSE and PSNR of the zonal codec for every r in [r_first, r_first + r_count)
    in one pass (config 5).  Returns (sse int64[batch, r_count], psnr float64[batch, r_count])."""
    import torch
    if images.dim() == 2:
        images = images.unsqueeze(0)
    n = images.shape[0]
    sse = torch.empty((n, r_count), dtype=torch.int64, device=images.device)
    psnr = torch.empty((n, r_count), dtype=torch.float64, device=images.device)
    dct16a_zonal_sweep(images, r_first, r_count, sse, psnr, desc_of(images, valid_height=valid_height), stream)
    return sse, psnr


def forward_host(host_images, host_coef, chunk_images=256, device=None, workspace=None, stream=None):
    """End-to-end forward transform from PINNED host images to PINNED host
    coefficients through the C entry dct16a_forward_host: chunks of
    `chunk_images` images alternate between two library streams, so the
    host->device copies, the transform and the device->host copies overlap.
    Returns the device workspace for reuse (pass it back as `workspace`).

    host_images: (batch, H, W) uint8/int16 pinned CPU tensor.
    host_coef:   (batch·H/16·W/16, 16, 16) int32 pinned CPU tensor.
    """
    import torch
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
    d = desc_of(host_images)
    need = dct16a_forward_host_workspace(d, chunk_images)
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(need, dtype=torch.uint8, device=dev)   # caching allocator: 512-B..2 MB aligned
        if workspace.data_ptr() % 1024:
            workspace = torch.empty(need + 1024, dtype=torch.uint8, device=dev)
            workspace = workspace[(-workspace.data_ptr()) % 1024:][:need]
    dct16a_forward_host(host_images, host_coef, workspace, d, stream)
    return workspace
