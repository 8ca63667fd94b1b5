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
        L.dct16a_forward16.argtypes = [vp, P(Desc), vp, vp]
        L.dct16a_forward16.restype = ctypes.c_int
        L.dct16a_ssim.argtypes = [vp, vp, P(Desc), vp, vp]
        L.dct16a_ssim.restype = ctypes.c_int
        L.dct16a_zonal_sweep.argtypes = [vp, P(Desc), ctypes.c_int32, ctypes.c_int32, vp, vp, vp]
        L.dct16a_zonal_sweep.restype = ctypes.c_int
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


def desc_of(images, bit_depth: int | None = None, valid_height: int | None = None) -> Desc:
    """Descriptor of a (batch, H, W) uint8 / int16 tensor (any strides with a
    unit inner stride)."""
    import torch
    if images.dim() == 2:
        images = images.unsqueeze(0)
    if bit_depth is None:
        bit_depth = 8 if images.dtype == torch.uint8 else 10
    elem = images.element_size()
    n, h, w = images.shape
    assert images.stride(2) == 1, "rows must be contiguous"
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


def _stream(stream):
    if stream is None:
        import torch
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


def dct16a_forward(src, coef, desc: Desc | None = None, stream=None) -> None:
    d = desc if desc is not None else desc_of(src)
    _check(lib().dct16a_forward(_ptr(src), ctypes.byref(d), _ptr(coef), _stream(stream)))


def dct16a_quantize(coef, qcoef, quant: Quant, desc: Desc, scaled=None, stream=None) -> None:
    _check(lib().dct16a_quantize(_ptr(coef), ctypes.byref(desc), ctypes.byref(quant), _ptr(qcoef),
                                 _ptr(scaled), _stream(stream)))


def dct16a_inverse(qcoef, recon, quant: Quant, desc: Desc, stream=None) -> None:
    _check(lib().dct16a_inverse(_ptr(qcoef), ctypes.byref(desc), ctypes.byref(quant), _ptr(recon),
                                _stream(stream)))


def dct16a_psnr(ref, test, sse, psnr=None, desc: Desc | None = None, stream=None) -> None:
    d = desc if desc is not None else desc_of(ref)
    _check(lib().dct16a_psnr(_ptr(ref), _ptr(test), ctypes.byref(d), _ptr(sse), _ptr(psnr), _stream(stream)))


def dct16a_codec(src, quant: Quant, sse, recon=None, psnr=None, desc: Desc | None = None, stream=None) -> None:
    d = desc if desc is not None else desc_of(src)
    _check(lib().dct16a_codec(_ptr(src), ctypes.byref(d), ctypes.byref(quant), _ptr(recon), _ptr(sse),
                              _ptr(psnr), _stream(stream)))


def dct16a_codec_allreduce(src, quant: Quant, sse_peers, frame_offset: int, recon=None, desc: Desc | None = None,
                           stream=None) -> None:
    """sse_peers: sequence of device addresses (ints) of every rank's int64 SSE
    vector, mapped into this device (e.g. torch symmetric memory buffer_ptrs)."""
    d = desc if desc is not None else desc_of(src)
    arr = (ctypes.c_void_p * len(sse_peers))(*[ctypes.c_void_p(int(a)) for a in sse_peers])
    _check(lib().dct16a_codec_allreduce(_ptr(src), ctypes.byref(d), ctypes.byref(quant), _ptr(recon), arr,
                                        len(sse_peers), int(frame_offset), _stream(stream)))


def dct16a_forward16(src, coef16, desc: Desc | None = None, stream=None) -> None:
    d = desc if desc is not None else desc_of(src)
    _check(lib().dct16a_forward16(_ptr(src), ctypes.byref(d), _ptr(coef16), _stream(stream)))


def dct16a_ssim(ref, test, ssim, desc: Desc | None = None, stream=None) -> None:
    d = desc if desc is not None else desc_of(ref)
    _check(lib().dct16a_ssim(_ptr(ref), _ptr(test), ctypes.byref(d), _ptr(ssim), _stream(stream)))


def dct16a_zonal_sweep(src, r_first: int, r_count: int, sse, psnr=None, desc: Desc | None = None,
                       stream=None) -> None:
    d = desc if desc is not None else desc_of(src)
    _check(lib().dct16a_zonal_sweep(_ptr(src), ctypes.byref(d), int(r_first), int(r_count), _ptr(sse), _ptr(psnr),
                                    _stream(stream)))


def dct16a_version() -> str:
    return lib().dct16a_version().decode()


def dct16a_last_error() -> str:
    return lib().dct16a_last_error().decode()


def dct16a_set_option(option: int, value: int) -> None:
    _check(lib().dct16a_set_option(option, value))


def dct16a_get_option(option: int) -> int:
    v = lib().dct16a_get_option(option)
    if option not in (OPT_CODEC_PATH, OPT_FWD_STORE):
        _check(v)
    return v
