"""ctypes binding of libdct16a.so (include/dct16a.h).

Argument marshalling only: every step of the path runs in the library's CUDA
kernels.  Tensors are torch CUDA tensors (PyTorch provides device memory and
streams); the stream defaults to torch's current stream.  There is no CPU
fallback: a missing library or a CPU tensor raises.
"""
from __future__ import annotations

import ctypes
import os

PKG = os.path.dirname(os.path.abspath(__file__))
# DCT16A_LIB overrides the library path (kernel-variant experiments under tools/)
LIB_PATH = os.environ.get("DCT16A_LIB") or os.path.join(PKG, "libdct16a.so")

ZONAL = 0
UNIFORM = 1
OPT_CODEC_PATH = 1
OPT_FWD_STORE = 2
OPT_UNIFORM_QUANT = 3

ERRORS = {-1: "ENULL", -2: "ESHAPE", -3: "EPITCH", -4: "EALIGN", -5: "EDOMAIN", -6: "ECUDA"}


class Dct16aError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"dct16a error {code} ({ERRORS.get(code, '?')}): {msg}")
        self.code = code


class Desc(ctypes.Structure):
    _fields_ = [("width", ctypes.c_int32), ("height", ctypes.c_int32),
                ("valid_height", ctypes.c_int32), ("batch", ctypes.c_int32),
                ("bit_depth", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("pitch_bytes", ctypes.c_int64), ("image_stride_bytes", ctypes.c_int64)]


class Quant(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int32), ("r", ctypes.c_int32), ("step", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


_lib = None


def lib() -> ctypes.CDLL:
    """Load libdct16a.so from the package directory (fails loudly if absent)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                               "(python -m paper_1606_05562_b200.build); there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        vp, P = ctypes.c_void_p, ctypes.POINTER
        L.dct16a_forward.argtypes = [vp, P(Desc), vp, vp]
        L.dct16a_quantize.argtypes = [vp, P(Desc), P(Quant), vp, vp, vp]
        L.dct16a_inverse.argtypes = [vp, P(Desc), P(Quant), vp, vp]
        L.dct16a_psnr.argtypes = [vp, vp, P(Desc), vp, vp, vp]
        L.dct16a_codec.argtypes = [vp, P(Desc), P(Quant), vp, vp, vp, vp]
        for f in ("dct16a_forward", "dct16a_quantize", "dct16a_inverse", "dct16a_psnr", "dct16a_codec"):
            getattr(L, f).restype = ctypes.c_int
        L.dct16a_codec_allreduce.argtypes = [vp, P(Desc), P(Quant), vp, P(vp), ctypes.c_int32, ctypes.c_int64, vp]
        L.dct16a_codec_allreduce.restype = ctypes.c_int
        L.dct16a_codec_allreduce_multicast.argtypes = [vp, P(Desc), P(Quant), vp, vp, ctypes.c_int64, vp]
        L.dct16a_codec_allreduce_multicast.restype = ctypes.c_int
        L.dct16a_forward16.argtypes = [vp, P(Desc), vp, vp]
        L.dct16a_forward16.restype = ctypes.c_int
        L.dct16a_ssim.argtypes = [vp, vp, P(Desc), vp, vp]
        L.dct16a_ssim.restype = ctypes.c_int
        L.dct16a_zonal_sweep.argtypes = [vp, P(Desc), ctypes.c_int32, ctypes.c_int32, vp, vp, vp]
        L.dct16a_zonal_sweep.restype = ctypes.c_int
        L.dct16a_sse_psnr.argtypes = [vp, ctypes.c_int64, P(Desc), vp, vp, vp, vp]
        L.dct16a_sse_psnr.restype = ctypes.c_int
        L.dct16a_forward_host.argtypes = [vp, P(Desc), vp, vp, ctypes.c_int64, vp]
        L.dct16a_forward_host.restype = ctypes.c_int
        L.dct16a_forward_host_workspace.argtypes = [P(Desc), ctypes.c_int32]
        L.dct16a_forward_host_workspace.restype = ctypes.c_int64
        L.dct16a_set_option.argtypes = [ctypes.c_int, ctypes.c_int]
        L.dct16a_set_option.restype = ctypes.c_int
        L.dct16a_get_option.argtypes = [ctypes.c_int]
        L.dct16a_get_option.restype = ctypes.c_int
        L.dct16a_last_error.restype = ctypes.c_char_p
        L.dct16a_version.restype = ctypes.c_char_p
        _lib = L
    return _lib


def _check(rc: int) -> None:
    if rc != 0:
        raise Dct16aError(rc, lib().dct16a_last_error().decode())


def make_desc(width: int, height: int, batch: int = 1, bit_depth: int = 8, pitch_bytes: int | None = None,
              image_stride_bytes: int | None = None, valid_height: int | None = None) -> Desc:
    elem = 1 if bit_depth == 8 else 2
    pitch = width * elem if pitch_bytes is None else pitch_bytes
    stride = pitch * height if image_stride_bytes is None else image_stride_bytes
    return Desc(width, height, height if valid_height is None else valid_height, batch, bit_depth, 0,
                pitch, stride)


def _pixel_depth(images, bit_depth):
    """The bit depth a pixel tensor's dtype admits: uint8 -> 8, int16/uint16 ->
    10 (values in [0, 1023]).  Any other dtype, or a bit depth its elements do
    not carry, raises (the kernels would read its bytes as pixels)."""
    import torch
    u16 = getattr(torch, "uint16", None)
    if images.dtype == torch.uint8:
        depth = 8
    elif images.dtype == torch.int16 or (u16 is not None and images.dtype == u16):
        depth = 10
    else:
        raise TypeError(f"pixels must be uint8 (8-bit) or int16/uint16 (10-bit), not {images.dtype}")
    if bit_depth is not None and int(bit_depth) != depth:
        raise ValueError(f"bit_depth {bit_depth} does not match pixel dtype {images.dtype}")
    return depth


def desc_of(images, bit_depth: int | None = None, valid_height: int | None = None) -> Desc:
    """Descriptor of a (batch, H, W) uint8 / int16 tensor (any strides with a
    unit inner stride)."""
    if images.dim() == 2:
        images = images.unsqueeze(0)
    if images.dim() != 3:
        raise ValueError("images must be (batch, H, W) or (H, W)")
    bit_depth = _pixel_depth(images, bit_depth)
    elem = images.element_size()
    n, h, w = images.shape
    if images.stride(2) != 1:
        raise ValueError("rows must be contiguous (unit inner stride)")
    return make_desc(w, h, n, bit_depth, images.stride(1) * elem, images.stride(0) * elem, valid_height)


def make_quant(mode: str | int = "zonal", r: int = 16, step: int = 16) -> Quant:
    m = {"zonal": ZONAL, "uniform": UNIFORM}.get(mode, mode)
    return Quant(int(m), int(r), int(step), 0)


def _ptr(t):
    if t is None:
        return None
    if hasattr(t, "is_cuda") and not t.is_cuda:
        raise ValueError("dct16a works on CUDA tensors only (no CPU fallback)")
    return ctypes.c_void_p(t.data_ptr())


def _n_blocks(d: Desc) -> int:
    return d.batch * (d.height // 16) * (d.width // 16)


def _need(t, name: str, numel: int, dtypes) -> None:
    """An output (or input) tensor must be contiguous with at least `numel`
    elements of one of `dtypes` (names of torch dtypes): the library writes
    that many elements through the raw pointer."""
    if t is None:
        return
    import torch
    ok = [getattr(torch, n) for n in dtypes if hasattr(torch, n)]
    if t.dtype not in ok:
        raise TypeError(f"{name} must be {'/'.join(dtypes)}, not {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if t.numel() < numel:
        raise ValueError(f"{name} has {t.numel()} elements, needs {numel}")


def _check_images(t, name: str, d: Desc) -> None:
    """A pixel tensor must hold the whole batch the descriptor describes."""
    if t is None:
        return
    _pixel_depth(t if t.dim() == 3 else t.unsqueeze(0), d.bit_depth)
    elem = 1 if d.bit_depth == 8 else 2
    extent = (d.batch - 1) * d.image_stride_bytes + (d.height - 1) * d.pitch_bytes + d.width * elem
    have = t.untyped_storage().nbytes() - t.storage_offset() * t.element_size()
    if have < extent:
        raise ValueError(f"{name}: descriptor spans {extent} bytes, tensor storage has {have}")


def _stream(stream):
    if stream is None:
        import torch
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


def dct16a_forward(src, coef, desc: Desc | None = None, stream=None) -> None:
    d = desc if desc is not None else desc_of(src)
    _check_images(src, "src", d)
    _need(coef, "coef", 256 * _n_blocks(d), ["int32"])
    _check(lib().dct16a_forward(_ptr(src), ctypes.byref(d), _ptr(coef), _stream(stream)))


def dct16a_quantize(coef, qcoef, quant: Quant, desc: Desc, scaled=None, stream=None) -> None:
    n = 256 * _n_blocks(desc)
    _need(coef, "coef", n, ["int32"])
    _need(qcoef, "qcoef", n, ["int32"])
    _need(scaled, "scaled", n, ["float32"])
    _check(lib().dct16a_quantize(_ptr(coef), ctypes.byref(desc), ctypes.byref(quant), _ptr(qcoef),
                                 _ptr(scaled), _stream(stream)))


def dct16a_inverse(qcoef, recon, quant: Quant, desc: Desc, stream=None) -> None:
    _need(qcoef, "qcoef", 256 * _n_blocks(desc), ["int32"])
    _check_images(recon, "recon", desc)
    _check(lib().dct16a_inverse(_ptr(qcoef), ctypes.byref(desc), ctypes.byref(quant), _ptr(recon),
                                _stream(stream)))


def dct16a_psnr(ref, test, sse, psnr=None, desc: Desc | None = None, stream=None) -> None:
    d = desc if desc is not None else desc_of(ref)
    _check_images(ref, "ref", d)
    _check_images(test, "test", d)
    _need(sse, "sse", d.batch, ["int64", "uint64"])
    _need(psnr, "psnr", d.batch, ["float64"])
    _check(lib().dct16a_psnr(_ptr(ref), _ptr(test), ctypes.byref(d), _ptr(sse), _ptr(psnr), _stream(stream)))


def dct16a_codec(src, quant: Quant, sse, recon=None, psnr=None, desc: Desc | None = None, stream=None) -> None:
    d = desc if desc is not None else desc_of(src)
    _check_images(src, "src", d)
    _check_images(recon, "recon", d)
    _need(sse, "sse", d.batch, ["int64", "uint64"])
    _need(psnr, "psnr", d.batch, ["float64"])
    _check(lib().dct16a_codec(_ptr(src), ctypes.byref(d), ctypes.byref(quant), _ptr(recon), _ptr(sse),
                              _ptr(psnr), _stream(stream)))


def dct16a_codec_allreduce(src, quant: Quant, sse_peers, frame_offset: int, recon=None, desc: Desc | None = None,
                           stream=None, multicast: bool = False) -> None:
    """sse_peers: sequence of device addresses (ints) of every rank's int64 SSE
    vector, mapped into this device (e.g. torch symmetric memory buffer_ptrs);
    multicast=True: sse_peers = [the NVLS multicast address of those vectors]
    (dct16a_codec_allreduce_multicast)."""
    d = desc if desc is not None else desc_of(src)
    _check_images(src, "src", d)
    _check_images(recon, "recon", d)
    if multicast:
        if len(sse_peers) != 1:
            raise ValueError("multicast takes exactly one address")
        _check(lib().dct16a_codec_allreduce_multicast(_ptr(src), ctypes.byref(d), ctypes.byref(quant), _ptr(recon),
                                                      ctypes.c_void_p(int(sse_peers[0])), int(frame_offset),
                                                      _stream(stream)))
        return
    arr = (ctypes.c_void_p * len(sse_peers))(*[ctypes.c_void_p(int(a)) for a in sse_peers])
    _check(lib().dct16a_codec_allreduce(_ptr(src), ctypes.byref(d), ctypes.byref(quant), _ptr(recon), arr,
                                        len(sse_peers), int(frame_offset), _stream(stream)))


def dct16a_forward16(src, coef16, desc: Desc | None = None, stream=None) -> None:
    d = desc if desc is not None else desc_of(src)
    _check_images(src, "src", d)
    _need(coef16, "coef16", 256 * _n_blocks(d), ["int16", "uint16"])
    _check(lib().dct16a_forward16(_ptr(src), ctypes.byref(d), _ptr(coef16), _stream(stream)))


def dct16a_ssim(ref, test, ssim, desc: Desc | None = None, stream=None) -> None:
    d = desc if desc is not None else desc_of(ref)
    _check_images(ref, "ref", d)
    _check_images(test, "test", d)
    _need(ssim, "ssim", d.batch, ["float64"])
    _check(lib().dct16a_ssim(_ptr(ref), _ptr(test), ctypes.byref(d), _ptr(ssim), _stream(stream)))


def dct16a_zonal_sweep(src, r_first: int, r_count: int, sse, psnr=None, desc: Desc | None = None,
                       stream=None) -> None:
    d = desc if desc is not None else desc_of(src)
    _check_images(src, "src", d)
    _need(sse, "sse", d.batch * int(r_count), ["int64", "uint64"])
    _need(psnr, "psnr", d.batch * int(r_count), ["float64"])
    _check(lib().dct16a_zonal_sweep(_ptr(src), ctypes.byref(d), int(r_first), int(r_count), _ptr(sse), _ptr(psnr),
                                    _stream(stream)))


def dct16a_sse_psnr(sse, count: int, desc: Desc, psnr=None, sse_total=None, psnr_total=None, stream=None) -> None:
    _need(sse, "sse", count, ["int64", "uint64"])
    _need(psnr, "psnr", count, ["float64"])
    _need(sse_total, "sse_total", 1, ["int64", "uint64"])
    _need(psnr_total, "psnr_total", 1, ["float64"])
    _check(lib().dct16a_sse_psnr(_ptr(sse), int(count), ctypes.byref(desc), _ptr(psnr), _ptr(sse_total),
                                 _ptr(psnr_total), _stream(stream)))


def dct16a_forward_host_workspace(desc: Desc, chunk_images: int) -> int:
    v = lib().dct16a_forward_host_workspace(ctypes.byref(desc), int(chunk_images))
    if v < 0:
        _check(int(v))
    return int(v)


def dct16a_forward_host(host_src, host_coef, workspace, desc: Desc | None = None, stream=None) -> None:
    """host_src / host_coef: CPU tensors (pinned for overlap); workspace: a
    CUDA uint8 tensor (1024-byte aligned, see dct16a_forward_host_workspace)."""
    d = desc if desc is not None else desc_of(host_src)
    for t, name in ((host_src, "host_src"), (host_coef, "host_coef")):
        if t.is_cuda:
            raise ValueError(f"{name} must be a host (CPU) tensor")
    _check_images(host_src, "host_src", d)
    _need(host_coef, "host_coef", 256 * _n_blocks(d), ["int32"])
    if not workspace.is_cuda:
        raise ValueError("workspace must be a CUDA tensor")
    _check(lib().dct16a_forward_host(ctypes.c_void_p(host_src.data_ptr()), ctypes.byref(d),
                                     ctypes.c_void_p(host_coef.data_ptr()), _ptr(workspace),
                                     workspace.numel() * workspace.element_size(), _stream(stream)))


def dct16a_version() -> str:
    return lib().dct16a_version().decode()


def dct16a_last_error() -> str:
    return lib().dct16a_last_error().decode()


def dct16a_set_option(option: int, value: int) -> None:
    _check(lib().dct16a_set_option(option, value))


def dct16a_get_option(option: int) -> int:
    v = lib().dct16a_get_option(option)
    if option not in (OPT_CODEC_PATH, OPT_FWD_STORE, OPT_UNIFORM_QUANT):
        _check(v)
    return v
