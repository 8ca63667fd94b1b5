"""C-ABI checks that need no GPU: the library loads, exports every symbol that
include/dct16a.h declares, and validates arguments synchronously (before any
CUDA call) with the documented error codes."""
import ctypes
import os
import re
import subprocess

import pytest

import paper_1606_05562_b200 as pkg
from paper_1606_05562_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "dct16a.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"DCT16A_API\s+[\w\s\*]*?\b(dct16a_\w+)\s*\(", text)))


def test_library_loads_and_exports_header_symbols():
    L = pkg.lib()
    syms = declared_symbols()
    assert len(syms) == 17
    for s in syms:
        assert hasattr(L, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (dct16a_\w+)", out))
    assert set(syms) <= exported
    # nothing but the ABI is exported from the dct16a namespace
    assert all(s.startswith("dct16a_") for s in exported)


def test_version():
    assert pkg.dct16a_version().startswith("dct16a ")
    assert "sm_100a" in pkg.dct16a_version()


def test_struct_layout_matches_header():
    assert ctypes.sizeof(_lib.Desc) == 40
    assert ctypes.sizeof(_lib.Quant) == 16


def _call_forward(desc, src=16, coef=16):
    L = pkg.lib()
    return L.dct16a_forward(ctypes.c_void_p(src), ctypes.byref(desc), ctypes.c_void_p(coef), None)


@pytest.mark.parametrize("kw,code", [
    (dict(width=0), -2), (dict(width=24), -2), (dict(height=-16), -2), (dict(batch=0), -2),
    (dict(valid_height=0), -2), (dict(valid_height=32), -2), (dict(bit_depth=12), -5),
    (dict(pitch_bytes=8), -3), (dict(pitch_bytes=72), -3), (dict(image_stride_bytes=8), -3),
])
def test_forward_validation_codes(kw, code):
    base = dict(width=64, height=16, valid_height=16, batch=2, bit_depth=8, pitch_bytes=64,
                image_stride_bytes=1024)
    base.update(kw)
    d = _lib.Desc(base["width"], base["height"], base["valid_height"], base["batch"], base["bit_depth"], 0,
                  base["pitch_bytes"], base["image_stride_bytes"])
    assert _call_forward(d) == code
    assert pkg.dct16a_last_error() != ""


def test_pointer_validation():
    d = _lib.make_desc(64, 16, 1, 8)
    assert _call_forward(d, src=0) == -1            # ENULL
    assert _call_forward(d, src=8) == -4            # EALIGN
    assert _call_forward(d, coef=4) == -4
    L = pkg.lib()
    assert L.dct16a_forward(ctypes.c_void_p(16), None, ctypes.c_void_p(16), None) == -1


@pytest.mark.parametrize("q,code", [
    (dict(mode=0, r=0), -5), (dict(mode=0, r=257), -5), (dict(mode=1, step=0), -5),
    (dict(mode=7), -5), (dict(mode=1, step=70000), -5)])
def test_quant_validation(q, code):
    d = _lib.make_desc(64, 16, 1, 8)
    qq = _lib.Quant(q.get("mode", 0), q.get("r", 16), q.get("step", 16), 0)
    L = pkg.lib()
    rc = L.dct16a_codec(ctypes.c_void_p(16), ctypes.byref(d), ctypes.byref(qq), None, ctypes.c_void_p(16),
                        None, None)
    assert rc == code
    rc = L.dct16a_quantize(ctypes.c_void_p(16), ctypes.byref(d), ctypes.byref(qq), ctypes.c_void_p(16),
                           None, None)
    assert rc == code


def test_codec_pointer_rules():
    d = _lib.make_desc(64, 16, 1, 8)
    q = _lib.make_quant("zonal", 16)
    L = pkg.lib()
    assert L.dct16a_codec(ctypes.c_void_p(16), ctypes.byref(d), ctypes.byref(q), None, None, None, None) == -1
    assert L.dct16a_codec(ctypes.c_void_p(16), ctypes.byref(d), ctypes.byref(q), None, ctypes.c_void_p(12),
                          None, None) == -4
    assert L.dct16a_codec(ctypes.c_void_p(32), ctypes.byref(d), ctypes.byref(q), ctypes.c_void_p(32),
                          ctypes.c_void_p(16), None, None) == -5   # recon aliases src


def test_binding_rejects_cpu_tensors():
    torch = pytest.importorskip("torch")
    x = torch.zeros((1, 16, 16), dtype=torch.uint8)
    with pytest.raises(ValueError):
        pkg.dct16a_forward(x, torch.zeros((1, 16, 16), dtype=torch.int32))


def test_options_validate_and_round_trip():
    """The product library ships codec paths 0/2 and forward store modes
    -1/3/5; the round-1 experiment variants (codec paths 1 and 3, store modes
    0-2, 4, 6, 7) exist only in -DDCT16A_EXPERIMENTS builds."""
    old = pkg.dct16a_get_option(pkg.OPT_CODEC_PATH)
    for v in (0, 2):
        pkg.dct16a_set_option(pkg.OPT_CODEC_PATH, v)
        assert pkg.dct16a_get_option(pkg.OPT_CODEC_PATH) == v
    pkg.dct16a_set_option(pkg.OPT_CODEC_PATH, old)
    for bad in (1, 3, 4, -1):
        with pytest.raises(pkg.Dct16aError) as e:
            pkg.dct16a_set_option(pkg.OPT_CODEC_PATH, bad)
        assert e.value.code == -5
    old = pkg.dct16a_get_option(pkg.OPT_FWD_STORE)
    for v in (-1, 3, 5):
        pkg.dct16a_set_option(pkg.OPT_FWD_STORE, v)
        assert pkg.dct16a_get_option(pkg.OPT_FWD_STORE) == v
    pkg.dct16a_set_option(pkg.OPT_FWD_STORE, old)
    for bad in (0, 1, 2, 4, 6, 7, 8):
        with pytest.raises(pkg.Dct16aError):
            pkg.dct16a_set_option(pkg.OPT_FWD_STORE, bad)
    old = pkg.dct16a_get_option(pkg.OPT_UNIFORM_QUANT)
    assert old == 0
    for v in (0, 1, 2):
        pkg.dct16a_set_option(pkg.OPT_UNIFORM_QUANT, v)
        assert pkg.dct16a_get_option(pkg.OPT_UNIFORM_QUANT) == v
    pkg.dct16a_set_option(pkg.OPT_UNIFORM_QUANT, old)
    for bad in (-1, 3):
        with pytest.raises(pkg.Dct16aError):
            pkg.dct16a_set_option(pkg.OPT_UNIFORM_QUANT, bad)
    with pytest.raises(pkg.Dct16aError) as e:
        pkg.dct16a_set_option(99, 0)
    assert e.value.code == -5


def test_library_is_the_trimmed_product_build():
    """The experiment kernels are not in the shipped library."""
    names = subprocess.run(["nm", "-C", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "fwd_kernel<1, 5>" in names and "codec_warp_kernel" in names and "zband_kernel" in names
    assert "zonal_tpb_kernel" not in names and "codec_kernel(" not in names
    assert "fwd_kernel<1, 0>" not in names and "fwd_kernel<1, 7>" not in names


def test_overlapping_buffers_rejected():
    """recon must not intersect src (not only recon == src), and coef must not
    intersect src: the TMA stores would overwrite input tiles not yet read."""
    L = pkg.lib()
    d = pkg.make_desc(64, 64, 2, 8)                     # 2 images of 4 KB
    q = pkg.make_quant("zonal", 16)
    src, sse = 1 << 20, 1 << 24
    for recon in (src + 16, src + 4096, src - 4096):
        assert L.dct16a_codec(ctypes.c_void_p(src), ctypes.byref(d), ctypes.byref(q), ctypes.c_void_p(recon),
                              ctypes.c_void_p(sse), None, None) == -5
    assert "overlaps" in pkg.dct16a_last_error()
    assert L.dct16a_forward(ctypes.c_void_p(src), ctypes.byref(d), ctypes.c_void_p(src + 8192 - 16), None) == -5
    peers = (ctypes.c_void_p * 1)(ctypes.c_void_p(sse))
    assert L.dct16a_codec_allreduce(ctypes.c_void_p(src), ctypes.byref(d), ctypes.byref(q), ctypes.c_void_p(src + 32),
                                    peers, 1, 0, None) == -5


def test_binding_checks_dtypes_and_sizes():
    torch = pytest.importorskip("torch")
    for bad in (torch.float32, torch.int32, torch.int64):
        with pytest.raises(TypeError):
            pkg.desc_of(torch.zeros((1, 16, 16), dtype=bad))
    with pytest.raises(ValueError):
        pkg.desc_of(torch.zeros((1, 16, 16), dtype=torch.uint8), bit_depth=10)
    assert pkg.desc_of(torch.zeros((2, 32, 48), dtype=torch.int16)).bit_depth == 10
    x = torch.zeros((1, 32, 32), dtype=torch.uint8)
    with pytest.raises(ValueError, match="needs 1024"):
        pkg.dct16a_forward(x, torch.zeros((3, 16, 16), dtype=torch.int32))
    with pytest.raises(TypeError):
        pkg.dct16a_forward(x, torch.zeros((4, 16, 16), dtype=torch.int64))
    with pytest.raises(ValueError, match="needs 2"):
        pkg.dct16a_codec(torch.zeros((2, 16, 16), dtype=torch.uint8), pkg.make_quant(), torch.zeros(1, dtype=torch.int64))
    with pytest.raises(ValueError, match="descriptor spans"):
        pkg.dct16a_forward(x, torch.zeros((4, 16, 16), dtype=torch.int32), pkg.make_desc(32, 32, 2, 8))


def test_sse_psnr_and_forward_host_validation():
    L = pkg.lib()
    d = pkg.make_desc(64, 64, 1, 8)
    buf = ctypes.c_void_p(1 << 20)
    assert L.dct16a_sse_psnr(None, 4, ctypes.byref(d), None, None, None, None) == -1
    assert L.dct16a_sse_psnr(buf, 0, ctypes.byref(d), None, None, None, None) == -2
    assert L.dct16a_sse_psnr(ctypes.c_void_p((1 << 20) + 4), 4, ctypes.byref(d), None, None, None, None) == -4
    d2 = pkg.make_desc(512, 512, 10, 8)
    need1 = L.dct16a_forward_host_workspace(ctypes.byref(d2), 1)
    assert need1 == 2 * (512 * 512 + 1024 * 1024)
    assert L.dct16a_forward_host_workspace(ctypes.byref(d2), 4) == 4 * need1
    assert L.dct16a_forward_host_workspace(ctypes.byref(d2), 0) == -5
    h = ctypes.c_void_p(1 << 30)
    assert L.dct16a_forward_host(None, ctypes.byref(d2), h, buf, need1, None) == -1
    assert L.dct16a_forward_host(h, ctypes.byref(d2), h, ctypes.c_void_p((1 << 20) + 16), need1, None) == -4
    assert L.dct16a_forward_host(h, ctypes.byref(d2), h, buf, need1 - 1, None) == -5
    assert "workspace" in pkg.dct16a_last_error()


def test_zonal_sweep_validation():
    import torch
    L = pkg.lib()
    d = pkg.make_desc(64, 64, 1, 8)
    buf = ctypes.c_void_p(1 << 20)          # aligned dummy pointers: validation fails before any use
    for r0, rc in [(0, 5), (1, 0), (250, 8), (-3, 4)]:
        assert L.dct16a_zonal_sweep(buf, ctypes.byref(d), r0, rc, buf, None, None) == -5
    assert L.dct16a_zonal_sweep(buf, ctypes.byref(d), 1, 256, None, None, None) == -1
    assert L.dct16a_zonal_sweep(buf, ctypes.byref(d), 1, 256, ctypes.c_void_p((1 << 20) + 4), None, None) == -4
    del torch


def test_forward16_rejects_10bit():
    L = pkg.lib()
    d = pkg.make_desc(64, 64, 1, 10)
    buf = ctypes.c_void_p(1 << 20)
    assert L.dct16a_forward16(buf, ctypes.byref(d), buf, None) == -5


def _build_c_demo():
    out = os.path.join(ROOT, "build", "c_api_demo")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    pkgdir = os.path.dirname(_lib.LIB_PATH)
    cuda_lib = "/usr/local/cuda/lib64"
    cmd = ["gcc", "-O2", "-std=c99", "-Wall", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
           os.path.join(ROOT, "examples", "c_api_demo.c"), "-L", pkgdir, "-ldct16a", "-L", cuda_lib, "-lcudart",
           "-lm", f"-Wl,-rpath,{pkgdir}:{cuda_lib}", "-o", out]
    return subprocess.run(cmd, capture_output=True, text=True), out


def test_c_api_demo_compiles_and_links():
    """The ABI is usable from plain C: the demo compiles against include/dct16a.h
    and links against libdct16a.so (tests/test_gpu_parity.py runs it)."""
    r, out = _build_c_demo()
    assert r.returncode == 0, r.stderr
    assert os.path.exists(out)


def test_codec_allreduce_validation():
    L = pkg.lib()
    d = pkg.make_desc(64, 64, 1, 8)
    q = pkg.make_quant("uniform", step=16)
    buf = ctypes.c_void_p(1 << 20)
    peers = (ctypes.c_void_p * 2)(ctypes.c_void_p(1 << 20), ctypes.c_void_p(2 << 20))
    f = L.dct16a_codec_allreduce
    assert f(buf, ctypes.byref(d), ctypes.byref(q), None, peers, 0, 0, None) == -5
    assert f(buf, ctypes.byref(d), ctypes.byref(q), None, peers, 9, 0, None) == -5
    assert f(buf, ctypes.byref(d), ctypes.byref(q), None, peers, 2, -1, None) == -5
    assert f(buf, ctypes.byref(d), ctypes.byref(q), None, None, 2, 0, None) == -1
    bad = (ctypes.c_void_p * 1)(ctypes.c_void_p((1 << 20) + 4))
    assert f(buf, ctypes.byref(d), ctypes.byref(q), None, bad, 1, 0, None) == -4
    m = L.dct16a_codec_allreduce_multicast
    assert m(buf, ctypes.byref(d), ctypes.byref(q), None, None, 0, None) == -1
    assert m(buf, ctypes.byref(d), ctypes.byref(q), None, ctypes.c_void_p((2 << 20) + 4), 0, None) == -4
    assert m(buf, ctypes.byref(d), ctypes.byref(q), None, ctypes.c_void_p(2 << 20), -1, None) == -5


def test_build_flags_keep_subnormals():
    """The zonal kernels read pixel integers from subnormal float products (and
    state it explicitly with PTX mul.rm.f32x2 without .ftz); the library build
    must not switch on flush-to-zero or fast math globally either."""
    from paper_1606_05562_b200 import build
    flags = " ".join(build.FLAGS)
    assert "fast_math" not in flags and "ftz=true" not in flags
    src = open(os.path.join(ROOT, "paper_1606_05562_b200", "csrc", "ptx.cuh")).read()
    assert "mul.rm.f32x2" in src and "mul.rm.ftz" not in src


def test_psnr_rejects_huge_valid_region():
    """dct16a_psnr indexes 16-byte chunks of one image in 32 bits: a valid
    region of 32 GiB or more is a shape error, raised before any launch."""
    L = pkg.lib()
    W, H = 1 << 20, 1 << 15
    d = _lib.Desc(W, H, H, 1, 8, 0, W, W * H)
    buf = ctypes.c_void_p(1 << 20)
    assert L.dct16a_psnr(buf, buf, ctypes.byref(d), buf, None, None) == -2
    assert "32 GiB" in pkg.dct16a_last_error()
