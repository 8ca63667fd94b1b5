"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs.  Bar: integer Z, quantised integer stages,
reconstructed pixels and SSE bit-exact; float32 scaled stages within 1e-5
relative (and exactly 0 where the oracle is 0); PSNR within 1e-3 dB.
"""
import math
import os

import numpy as np
import pytest

import synth
from oracle import codec as oc

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1606_05562_b200 as pkg  # noqa: E402

DEV = torch.device("cuda:0")


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def oracle_Z(imgs):
    return oc.forward(oc.to_blocks(imgs.astype(np.int64))).reshape(-1, 16, 16)


def gpu_Z(imgs_t, desc=None):
    n, h, w = imgs_t.shape
    out = torch.empty((n * (h // 16) * (w // 16), 16, 16), dtype=torch.int32, device=DEV)
    pkg.dct16a_forward(imgs_t, out, desc if desc is not None else pkg.desc_of(imgs_t))
    torch.cuda.synchronize()
    return out.cpu().numpy()


def u8_cases():
    yield "cfg1", synth.image_u8(0)[None]
    yield "adversarial", synth.adversarial_u8(64, 64)
    yield "ragged17x3", synth.batch_u8([5, 6, 7], 48, 272)         # BX=17: tile of 32 is ragged
    yield "wide", synth.batch_u8([8], 32, 1920)                    # 120 blocks: 3 full tiles + 24
    yield "tiny", synth.batch_u8([9], 16, 16)
    yield "narrow", synth.batch_u8([10, 11], 64, 48)
    rng = np.random.default_rng(3)
    yield "uniform-noise", rng.integers(0, 256, size=(4, 64, 96)).astype(np.uint8)


@pytest.mark.parametrize("name,imgs", list(u8_cases()), ids=lambda v: v if isinstance(v, str) else "")
def test_forward_u8_bit_exact(name, imgs):
    assert np.array_equal(gpu_Z(to_dev(imgs)), oracle_Z(imgs))


@pytest.mark.parametrize("name,imgs", list(u8_cases()), ids=lambda v: v if isinstance(v, str) else "")
def test_forward16_bit_exact(name, imgs):
    """dct16a_forward16: the low 16 bits of Z (DC as uint16, AC as int16)."""
    x = to_dev(imgs)
    got = pkg.forward16(x).cpu().numpy().astype(np.int64)
    Z = oracle_Z(imgs)
    want = Z.copy()
    want[:, 0, 0] = Z[:, 0, 0] - 65536 * (Z[:, 0, 0] >= 32768)   # uint16 bits read as int16
    assert np.array_equal(got, want)
    assert np.all(np.abs(Z[:, 1:, :]) <= 32767) and np.all(np.abs(Z[:, 0, 1:]) <= 32767)


def test_forward_10bit_bit_exact():
    imgs = synth.frames_10bit([0, 1], H=64, W=272, workers=1)
    adv = synth.adversarial_u8(48, 80, bit_depth=10)
    for x in (imgs, adv):
        assert np.array_equal(gpu_Z(to_dev(x)), oracle_Z(x))


def test_forward_pitched_and_strided():
    big = synth.batch_u8([12, 13, 14], 80, 400)
    t = to_dev(big)[:, 8:72, 32:288]                   # pitch 400 > width 256, stride 32000
    view = big[:, 8:72, 32:288]
    assert np.array_equal(gpu_Z(t), oracle_Z(view))
    f = synth.frames_10bit([3], H=48, W=320, workers=1)
    t10 = to_dev(f)[:, :, 16:240]
    assert np.array_equal(gpu_Z(t10), oracle_Z(f[:, :, 16:240]))


def _quant_run(imgs, q, bit_depth):
    x = to_dev(imgs)
    d = pkg.desc_of(x, bit_depth)
    n, h, w = imgs.shape
    nb = n * (h // 16) * (w // 16)
    coef = torch.empty((nb, 16, 16), dtype=torch.int32, device=DEV)
    qc = torch.empty_like(coef)
    sc = torch.empty((nb, 16, 16), dtype=torch.float32, device=DEV)
    rec = torch.empty_like(x)
    pkg.dct16a_forward(x, coef, d)
    pkg.dct16a_quantize(coef, qc, q, d, sc)
    pkg.dct16a_inverse(qc, rec, q, d)
    torch.cuda.synchronize()
    return coef.cpu().numpy(), qc.cpu().numpy(), sc.cpu().numpy(), rec.cpu().numpy()


def _check_scaled(got, want, exact_int):
    """float32 stage vs the oracle's float64 dense product.  Zero-ness is
    decided on the oracle's exact integer stage (the float64 product of a zero
    coefficient carries ~1e-14 of rounding); elsewhere |rel| <= 1e-5."""
    want = want.reshape(got.shape)
    zero = exact_int.reshape(got.shape) == 0
    assert np.all(got[zero] == 0)
    assert np.all(np.abs(want[zero]) < 1e-9)
    rel = np.abs(got[~zero] - want[~zero]) / np.abs(want[~zero])
    assert rel.max() <= 1e-5, rel.max()


@pytest.mark.parametrize("r", [1, 2, 15, 16, 17, 32, 64, 128, 255, 256])
def test_zonal_stages_and_inverse(r):
    imgs = np.concatenate([synth.batch_u8([20, 21], 64, 64), synth.adversarial_u8(64, 64)])
    q = pkg.make_quant("zonal", r)
    Z, qc, sc, rec = _quant_run(imgs, q, 8)
    X = oc.to_blocks(imgs.astype(np.int64))
    ref = oc.zonal_codec(X, r)
    assert np.array_equal(Z, ref["Z"].reshape(Z.shape))
    assert np.array_equal(qc, ref["Zm"].reshape(qc.shape))
    _check_scaled(sc, ref["scaled"], ref["Zm"])
    assert np.array_equal(rec, oc.from_blocks(ref["recon"]))
    if r == 256:
        assert np.array_equal(rec, imgs)


@pytest.mark.parametrize("step", [1, 5, 16, 64])
def test_uniform_stages_and_inverse(step):
    imgs = np.concatenate([synth.frames_10bit([4, 5], H=64, W=96, workers=1),
                           synth.adversarial_u8(64, 96, bit_depth=10)])
    q = pkg.make_quant("uniform", step=step)
    Z, qc, sc, rec = _quant_run(imgs, q, 10)
    X = oc.to_blocks(imgs.astype(np.int64))
    ref = oc.uniform_codec(X, step, 10)
    assert np.array_equal(Z, ref["Z"].reshape(Z.shape))
    assert np.array_equal(qc, ref["q"].reshape(qc.shape))
    _check_scaled(sc, ref["scaled"], ref["Z"])
    assert np.array_equal(rec, oc.from_blocks(ref["recon"]))


def test_uniform_forced_ties():
    # coefficients exactly on a rounding tie in the rational cells must round away
    T = np.array(oc.T)
    g = np.diag(T @ T.T)
    Zs = np.zeros((1, 16, 16), dtype=np.int32)
    want = np.zeros((1, 16, 16), dtype=np.int64)
    step = 16
    rng = np.random.default_rng(0)
    for k in range(16):
        for l in range(16):
            G = int(g[k] * g[l])
            r = math.isqrt(G)
            m = int(rng.integers(0, 400))
            s = 1 if rng.random() < 0.5 else -1
            if r * r == G:
                z = (2 * m + 1) * step * r // 2
            else:
                z = int(rng.integers(0, 200000))
            Zs[0, k, l] = s * z
    want = oc.uniform_q(Zs.astype(np.int64), step)
    coef = to_dev(Zs)
    qc = torch.empty_like(coef)
    d = pkg.make_desc(16, 16, 1, 10)
    pkg.dct16a_quantize(coef, qc, pkg.make_quant("uniform", step=step), d)
    torch.cuda.synchronize()
    assert np.array_equal(qc.cpu().numpy(), want)


def test_psnr_kernel():
    a = synth.batch_u8([30, 31, 32], 64, 80)
    b = a.copy()
    b[0] ^= 1
    b[1, 40:, :] = 0
    x, y = to_dev(a), to_dev(b)
    sse = torch.empty(3, dtype=torch.int64, device=DEV)
    ps = torch.empty(3, dtype=torch.float64, device=DEV)
    pkg.dct16a_psnr(x, y, sse, ps)
    torch.cuda.synchronize()
    want = oc.sse(a, b)
    assert sse.cpu().tolist() == want
    for got, s in zip(ps.cpu().tolist(), want):
        exp = oc.psnr_from_sse(s, 64 * 80, 8)
        assert (math.isinf(got) and math.isinf(exp)) or abs(got - exp) < 1e-3
    # valid_height excludes rows
    d = pkg.desc_of(x, valid_height=32)
    pkg.dct16a_psnr(x, y, sse, ps, desc=d)
    torch.cuda.synchronize()
    assert sse.cpu().tolist() == oc.sse(a, b, 32)


@pytest.fixture(params=[0, 2], ids=["auto", "warp"])
def codec_path(request):
    """Every fused-codec test runs on each kernel choice of the product build
    (DCT16A_OPT_CODEC_PATH): the automatic choice (band-pruned warp-per-tile
    kernel for every zonal case) and the warp-per-block-pair kernel for
    everything, each checked against the oracle independently."""
    old = pkg.dct16a_get_option(pkg.OPT_CODEC_PATH)
    pkg.dct16a_set_option(pkg.OPT_CODEC_PATH, request.param)
    yield request.param
    pkg.dct16a_set_option(pkg.OPT_CODEC_PATH, old)


def _codec_check(imgs, mode, bit_depth, r=16, step=16, valid_height=None):
    x = to_dev(imgs)
    rec, sse, ps = pkg.codec(x, mode, r=r, step=step, valid_height=valid_height)
    torch.cuda.synchronize()
    ref = oc.codec_images(imgs, mode, r=r, step=step, bit_depth=bit_depth, valid_height=valid_height)
    assert np.array_equal(rec.cpu().numpy(), ref["recon_img"])
    assert sse.cpu().tolist() == ref["sse"]
    for got, exp in zip(ps.cpu().tolist(), ref["psnr"]):
        assert (math.isinf(got) and math.isinf(exp)) or abs(got - exp) < 1e-3
    return rec


def test_codec_config1(codec_path):
    _codec_check(synth.image_u8(0)[None], "zonal", 8, r=16)


@pytest.mark.parametrize("r", [1, 2, 10, 11, 16, 21, 22, 32, 36, 37, 100, 256])
def test_codec_zonal_varied(r, codec_path):
    # automatic choice: the band kernel on the smallest band holding r (r > 136: band 15, unpruned)
    imgs = np.concatenate([synth.batch_u8([40, 41], 48, 272), synth.adversarial_u8(48, 272)])
    _codec_check(imgs, "zonal", 8, r=r)


@pytest.mark.parametrize("shape", [(1, 16, 16), (3, 32, 48), (2, 64, 1920), (1, 48, 784)])
def test_codec_zonal_shapes(shape, codec_path):
    n, h, w = shape
    imgs = synth.batch_u8(range(60, 60 + n), h, w)
    for r in (16, 32):
        _codec_check(imgs, "zonal", 8, r=r)


def test_codec_zonal_padded_valid_height(codec_path):
    v = synth.video_u8(3, H=56, W=96, pad_to=64, workers=1)
    _codec_check(v, "zonal", 8, r=32, valid_height=56)


def test_codec_uniform(codec_path):
    f = np.concatenate([synth.frames_10bit([6, 7], H=64, W=128, workers=1),
                        synth.adversarial_u8(64, 128, bit_depth=10)])
    _codec_check(f, "uniform", 10, step=16)


def test_codec_equals_chain(codec_path):
    imgs = synth.batch_u8([50, 51], 64, 64)
    for mode, r, step, bd, src in [("zonal", 16, 16, 8, imgs),
                                   ("uniform", 16, 16, 10, synth.frames_10bit([8], H=64, W=64, workers=1))]:
        q = pkg.make_quant(mode, r, step)
        _, _, _, rec_chain = _quant_run(src, q, bd)
        rec = _codec_check(src, mode, bd, r=r, step=step)
        assert np.array_equal(rec.cpu().numpy(), rec_chain)


def test_codec_without_recon_output(codec_path):
    img = synth.image_u8(1)[None]
    x = to_dev(img)
    _, sse, ps = pkg.codec(x, "zonal", r=16, want_recon=False)
    torch.cuda.synchronize()
    assert sse.cpu().tolist() == oc.codec_images(img, "zonal", r=16)["sse"]
    f = synth.frames_10bit([12], H=48, W=208, workers=1)
    _, sse, ps = pkg.codec(to_dev(f), "uniform", step=16, want_recon=False)
    torch.cuda.synchronize()
    assert sse.cpu().tolist() == oc.codec_images(f, "uniform", step=16, bit_depth=10)["sse"]


@pytest.fixture(params=[0, 1, 2], ids=["quant-auto", "quant-float", "quant-fixed"])
def uniform_quant(request):
    """Every uniform case on each quantiser choice (DCT16A_OPT_UNIFORM_QUANT):
    automatic, always float32, fixed point wherever its bound allows."""
    old = pkg.dct16a_get_option(pkg.OPT_UNIFORM_QUANT)
    pkg.dct16a_set_option(pkg.OPT_UNIFORM_QUANT, request.param)
    yield request.param
    pkg.dct16a_set_option(pkg.OPT_UNIFORM_QUANT, old)


@pytest.mark.parametrize("step", [1, 2, 3, 4, 5, 6, 7, 10, 16, 24, 100, 200, 65535])
def test_codec_uniform_quantiser_choices(step, uniform_quant):
    """Both uniform quantisers (and the automatic choice) give the oracle's
    bytes on 10-bit frames and 8-bit images, ragged shapes, small to huge steps."""
    f = synth.frames_10bit([40, 41], H=48, W=208, workers=1)
    _codec_check(f, "uniform", 10, step=step)
    u8 = synth.batch_u8(range(42, 44), 48, 208)
    _codec_check(u8, "uniform", 8, step=step)


@pytest.mark.parametrize("step", [1, 2, 3, 4, 5, 6, 7, 16, 24, 200, 65535])
@pytest.mark.parametrize("shape", [(1, 16, 16), (2, 48, 208), (1, 32, 1920)])
def test_codec_uniform_steps_and_shapes(step, shape, codec_path):
    """Uniform codec (warp kernel) for small to huge steps — Δ <= 6 takes the
    fixed-point quantiser, larger steps the float one — a single block, a
    ragged tile (13 blocks per strip) and a wide strip, 10-bit and 8-bit."""
    n, h, w = shape
    f = synth.frames_10bit(list(range(20, 20 + n)), H=h, W=w, workers=1)
    _codec_check(f, "uniform", 10, step=step)
    u8 = synth.batch_u8(range(30, 30 + n), h, w)
    _codec_check(u8, "uniform", 8, step=step)


@pytest.mark.parametrize("r", [1, 16, 37, 100, 256])
def test_codec_zonal_10bit(r, codec_path):
    f = np.concatenate([synth.frames_10bit([14, 15], H=48, W=208, workers=1),
                        synth.adversarial_u8(48, 208, bit_depth=10)])
    _codec_check(f, "zonal", 10, r=r)


def _tie_levels():
    """Levels with exact .5 ties of the reconstruction (irrational parts
    cancelled: only rational cells g_k = g_l populated) and near-ties, with
    the steps that produce them (oracle pins: test_uniform_recon_exact_ties_*)."""
    T = np.array(oc.T)
    g = np.diag(T @ T.T)
    rational = np.array([[g[k] == g[l] for l in range(16)] for k in range(16)])
    rng = np.random.default_rng(17)
    cases = []
    q = np.zeros((4, 16, 16), dtype=np.int32)
    q[0, 0, 0] = 1                                  # Δ=24: 1.5 everywhere
    q[1, 0, 0], q[1, 2, 2] = 8, 1                   # Δ=6: 3 ± 1/2
    q[2] = rng.integers(-3, 4, size=(16, 16)) * rational
    q[2, 0, 0] = 40
    q[3] = rng.integers(-2, 3, size=(16, 16))
    q[3, 0, 0] = 60
    for step in (24, 6, 12, 16):
        cases.append((step, q.copy()))
    r = rng.integers(-3, 4, size=(64, 16, 16)).astype(np.int32) * rational
    r[:, 0, 0] = rng.integers(20, 90, size=64)
    cases.append((6, r))
    return cases


@pytest.mark.parametrize("case", range(5))
def test_uniform_inverse_exact_ties(case):
    """dct16a_inverse (uniform) on levels whose reconstruction has exact .5
    ties or near-ties: pixels must equal the oracle's exact decisions."""
    step, q = _tie_levels()[case]
    nb = q.shape[0]
    want = oc.uniform_inverse_levels(q.astype(np.int64), step, bit_depth=10)
    if step in (24, 6):
        assert want["n_near_ties"] > 0
    qd = to_dev(q.reshape(nb, 16, 16))
    rec = torch.zeros((1, 16, 16 * nb), dtype=torch.int16, device=DEV)
    pkg.dct16a_inverse(qd, rec, pkg.make_quant("uniform", step=step), pkg.desc_of(rec, 10))
    torch.cuda.synchronize()
    got = rec.cpu().numpy()[0].reshape(16, nb, 16).transpose(1, 0, 2)
    assert np.array_equal(got, want["recon"])


# ------------------------------------------------- full-size configurations
@pytest.mark.slow
def test_config2_full_size_sampled():
    """Config 2 at full size (4096 x 512² u8) in the launch configuration that
    bench.py times: sampled blocks checked against the oracle one by one, and
    properties that hold for every block checked on all 4.19M blocks."""
    n = 4096
    imgs = synth.batch_u8(range(n), 512, 512)
    x = to_dev(imgs)
    coef = pkg.forward(x)
    torch.cuda.synchronize()
    rng = np.random.default_rng(2)
    idx = rng.choice(coef.shape[0], size=3000, replace=False)
    got = coef[torch.from_numpy(idx).to(DEV)].cpu().numpy()
    Xb = oc.to_blocks(imgs.astype(np.int64)).reshape(-1, 16, 16)
    assert np.array_equal(got, oc.forward(Xb[idx]))
    # every block: DC = block sum, integer Parseval sum W·Z² = 2304·sum X²
    T = np.array(oc.T)
    g = np.diag(T @ T.T)
    W = torch.from_numpy((2304 // np.outer(g, g)).astype(np.int64)).to(DEV)
    for s in range(0, coef.shape[0], 1 << 20):
        z = coef[s:s + (1 << 20)].to(torch.int64)
        xb = x.view(n, 32, 16, 32, 16).permute(0, 1, 3, 2, 4).reshape(-1, 16, 16)[s:s + (1 << 20)].to(torch.int64)
        assert torch.equal(z[:, 0, 0], xb.sum(dim=(1, 2)))
        assert torch.equal((W * z * z).sum(dim=(1, 2)), 2304 * (xb * xb).sum(dim=(1, 2)))


@pytest.mark.slow
def test_config4_full_size_tiled():
    """Config 4 geometry at full size — 1000 frames of 3840x2160 int16 (16.6 GB,
    so every offset past frame 258 needs 64 bits) — through dct16a_codec in the
    launch configuration tools/bench_configs.py times.  The frames repeat 8
    distinct generated frames; every per-frame SSE and the recon of sampled
    frames (first, middle, last) are checked against the oracle."""
    k = 8
    src = synth.frames_10bit(range(k))
    sd = to_dev(src)
    n = 1000
    x = torch.empty((n, 2160, 3840), dtype=torch.int16, device=DEV)
    for f in range(n):
        x[f].copy_(sd[f % k])
    rec, sse, ps = pkg.codec(x, "uniform", step=16)
    torch.cuda.synchronize()
    refs = [oc.codec_images(src[i:i + 1], "uniform", step=16, bit_depth=10) for i in range(k)]
    got_sse = sse.cpu().tolist()
    assert got_sse == [refs[f % k]["sse"][0] for f in range(n)]
    for f in (0, 1, 517, n - 1):
        assert np.array_equal(rec[f].cpu().numpy(), refs[f % k]["recon_img"][0]), f
    for f in (0, n - 1):
        assert abs(float(ps[f]) - refs[f % k]["psnr"][0]) < 1e-3


@pytest.mark.slow
def test_config3_full_size_sampled():
    """Config 3 at full size (600 x 1920x1088 padded video, zonal r = 32,
    PSNR over the 1080 visible rows) in the bench launch configuration;
    sampled frames checked against the oracle."""
    v = synth.video_u8(600)
    x = to_dev(v)
    rec, sse, ps = pkg.codec(x, "zonal", r=32, valid_height=1080)
    torch.cuda.synchronize()
    got_sse = sse.cpu().tolist()
    for f in (0, 1, 299, 598, 599):
        ref = oc.codec_images(v[f:f + 1], "zonal", r=32, valid_height=1080)
        assert np.array_equal(rec[f].cpu().numpy(), ref["recon_img"][0]), f
        assert got_sse[f] == ref["sse"][0]
        assert abs(float(ps[f]) - ref["psnr"][0]) < 1e-3


@pytest.mark.parametrize("frames", [24])
def test_codec_mid_size_claim_runs(frames):
    """Mid-size launches, where the tile claims are shorter than the default
    run (2-5 tiles for the band kernel, 3-4 for the warp kernel): every frame's
    SSE and every reconstruction against the oracle, zonal and uniform."""
    v = synth.video_u8(frames)
    x = to_dev(v)
    for mode in ("zonal", "uniform"):
        rec, sse, _ = pkg.codec(x, mode, r=32, step=16, valid_height=1080)
        torch.cuda.synchronize()
        ref = oc.codec_images(v, mode, r=32, step=16, valid_height=1080)
        assert np.array_equal(rec.cpu().numpy(), ref["recon_img"]), mode
        assert sse.cpu().tolist() == ref["sse"], mode


# ------------------------------------------------------ config 5: r-sweep
def _sweep_check(imgs, bd, r_first, r_count, valid_height=None):
    x = to_dev(imgs)
    sse, ps = pkg.zonal_sweep(x, r_first, r_count, valid_height=valid_height)
    torch.cuda.synchronize()
    got = sse.cpu().numpy()
    gps = ps.cpu().numpy()
    for i, r in enumerate(range(r_first, r_first + r_count)):
        ref = oc.codec_images(imgs, "zonal", r=r, bit_depth=bd, valid_height=valid_height)
        assert got[:, i].tolist() == ref["sse"], r
        for a, b in zip(gps[:, i].tolist(), ref["psnr"]):
            assert (math.isinf(a) and math.isinf(b)) or abs(a - b) < 1e-3
    return got


@pytest.mark.parametrize("bd", [8, 10])
def test_zonal_sweep_every_r(bd):
    """dct16a_zonal_sweep: SSE and PSNR for every r = 1..256 equal the oracle's
    zonal codec with that r (ragged tile, adversarial blocks, 8/10-bit)."""
    if bd == 8:
        imgs = np.concatenate([synth.batch_u8([70, 71], 48, 208), synth.adversarial_u8(48, 208)])
    else:
        imgs = np.concatenate([synth.frames_10bit([16], H=48, W=208, workers=1),
                               synth.adversarial_u8(48, 208, bit_depth=10)])
    got = _sweep_check(imgs, bd, 1, 256)
    assert np.all(got[:, -1] == 0)                       # r = 256 is lossless


def test_zonal_sweep_subrange_and_valid_height(codec_path):
    v = synth.video_u8(2, H=40, W=272, pad_to=48, workers=1)
    got = _sweep_check(v, 8, 30, 40, valid_height=40)
    # and the same numbers from the fused codec, r by r
    x = to_dev(v)
    for i, r in enumerate((30, 36, 37, 69)):
        _, sse, _ = pkg.codec(x, "zonal", r=r, valid_height=40, want_recon=False)
        torch.cuda.synchronize()
        assert sse.cpu().tolist() == got[:, r - 30].tolist()


@pytest.mark.slow
def test_config5_full_size_sampled():
    """Config 5 at full size (64 x 1024² images, r = 1..256 in one sweep):
    every r of one image per rho group against the oracle."""
    imgs = synth.config5_images()
    x = to_dev(imgs)
    sse, ps = pkg.zonal_sweep(x, 1, 256)
    torch.cuda.synchronize()
    got = sse.cpu().numpy()
    assert np.all(got[:, 255] == 0)
    # SSIM of the r = 16 reconstructions (the paper's second measure)
    rec, _, _ = pkg.codec(x, "zonal", r=16)
    ss = pkg.ssim(x, rec).cpu().numpy()
    recn = rec.cpu().numpy()
    for n in (0, 16, 32, 48):
        assert abs(ss[n] - oq.ssim(imgs[n:n + 1], recn[n:n + 1])[0]) < 1e-9
    for n in (0, 16, 32, 48):
        img = imgs[n:n + 1]
        X = oc.to_blocks(img.astype(np.int64))
        Z = oc.forward(X)
        for r in range(1, 257):
            N = oc.zonal_numerator(oc.zonal_stage(Z, r))
            rec = oc.clamp_pixels(oc.round_half_away_rational(N, 2304), 8)
            assert int(got[n, r - 1]) == oc.sse(img, oc.from_blocks(rec))[0], (n, r)


def test_config4_sharded_runner_torchrun():
    """tools/run_config4.py under torchrun (NCCL process group, one rank on
    this box): sharding + codec + SSE all-reduce give the oracle's per-frame
    SSE and global PSNR."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
           "--master-addr=127.0.0.1", "--master-port=29533", os.path.join(root, "tools", "run_config4.py"),
           "--frames", "5", "--height", "64", "--width", "208", "--reps", "1", "--dump", "--fused"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    f = synth.frames_10bit(range(5), H=64, W=208, workers=1)
    ref = oc.codec_images(f, "uniform", step=16, bit_depth=10)
    assert line["sse"] == ref["sse"]
    # the in-kernel all-reduce over symmetric memory (dct16a_codec_allreduce) agrees
    assert line["fused_allreduce"]["equal_to_nccl"] is True
    P = 5 * 64 * 208
    assert abs(line["global_psnr_db"] - oc.psnr_from_sse(sum(ref["sse"]), P, 10)) < 1e-9


# ----------------------------------------------------------------- SSIM
from oracle import quality as oq  # noqa: E402


def test_ssim_kernel_against_oracle():
    """dct16a_ssim (float64, Wang 2004 defaults) against the oracle's plain
    sliding-window SSIM: codec reconstructions, 10-bit, valid_height, ragged
    widths, identical and negated images; |Δ| <= 1e-9."""
    imgs = np.concatenate([synth.batch_u8([80, 81], 48, 208), synth.adversarial_u8(48, 208)])
    x = to_dev(imgs)
    rec, _, _ = pkg.codec(x, "zonal", r=16)
    torch.cuda.synchronize()
    got = pkg.ssim(x, rec).cpu().numpy()
    want = oq.ssim(imgs, rec.cpu().numpy())
    assert np.max(np.abs(got - want)) < 1e-9
    assert np.all(pkg.ssim(x, x).cpu().numpy() == 1.0)
    neg = to_dev(255 - imgs)
    assert np.max(np.abs(pkg.ssim(x, neg).cpu().numpy() - oq.ssim(imgs, 255 - imgs))) < 1e-9
    f = synth.frames_10bit([21, 22], H=64, W=144, workers=1)
    fd = to_dev(f)
    fr, _, _ = pkg.codec(fd, "uniform", step=16)
    torch.cuda.synchronize()
    assert np.max(np.abs(pkg.ssim(fd, fr).cpu().numpy() - oq.ssim(f, fr.cpu().numpy(), 10))) < 1e-9
    v = synth.video_u8(2, H=40, W=96, pad_to=48, workers=1)
    vd = to_dev(v)
    vr, _, _ = pkg.codec(vd, "zonal", r=32, valid_height=40)
    torch.cuda.synchronize()
    got = pkg.ssim(vd, vr, valid_height=40).cpu().numpy()
    assert np.max(np.abs(got - oq.ssim(v, vr.cpu().numpy(), valid_height=40))) < 1e-9
    t = synth.batch_u8([83], 16, 16)
    td = to_dev(t)
    tr_, _, _ = pkg.codec(td, "zonal", r=4)
    torch.cuda.synchronize()
    assert abs(float(pkg.ssim(td, tr_)[0]) - oq.ssim(t, tr_.cpu().numpy())[0]) < 1e-9


@pytest.mark.slow
def test_ssim_config1_and_config5_sample():
    img = synth.image_u8(0)[None]
    x = to_dev(img)
    rec, _, _ = pkg.codec(x, "zonal", r=16)
    torch.cuda.synchronize()
    got = float(pkg.ssim(x, rec)[0])
    assert abs(got - oq.ssim(img, rec.cpu().numpy())[0]) < 1e-9
    assert 0.5 < got < 1.0


def test_pitched_strided_views_every_entry(codec_path):
    """Views with row pitch > width and image stride > pitch·height (a window
    of larger images): forward16, the fused codec (zonal and uniform), the
    r-sweep and SSIM must see exactly the window."""
    big = synth.batch_u8([90, 91], 80, 400)
    view = big[:, 8:72, 32:288]                     # pitch 400, stride 32000, 256 x 64 window
    t = to_dev(big)[:, 8:72, 32:288]
    vw = np.ascontiguousarray(view)
    Z = oracle_Z(vw)
    got16 = pkg.forward16(t).cpu().numpy().astype(np.int64)
    Z16 = Z.copy()
    Z16[:, 0, 0] = Z[:, 0, 0] - 65536 * (Z[:, 0, 0] >= 32768)
    assert np.array_equal(got16, Z16)
    for mode, r, step, bd, src_big, win in [("zonal", 32, 16, 8, big, (slice(8, 72), slice(32, 288))),
                                            ("zonal", 60, 16, 8, big, (slice(8, 72), slice(32, 288)))]:
        x = to_dev(src_big)[:, win[0], win[1]]
        rec, sse, _ = pkg.codec(x, mode, r=r, step=step)
        torch.cuda.synchronize()
        ref = oc.codec_images(np.ascontiguousarray(src_big[:, win[0], win[1]]), mode, r=r, step=step, bit_depth=bd)
        assert np.array_equal(rec.cpu().numpy(), ref["recon_img"])
        assert sse.cpu().tolist() == ref["sse"]
    f = synth.frames_10bit([30, 31], H=80, W=272, workers=1)
    fv = np.ascontiguousarray(f[:, 16:64, 16:208])
    ft = to_dev(f)[:, 16:64, 16:208]
    rec, sse, _ = pkg.codec(ft, "uniform", step=16)
    torch.cuda.synchronize()
    ref = oc.codec_images(fv, "uniform", step=16, bit_depth=10)
    assert np.array_equal(rec.cpu().numpy(), ref["recon_img"])
    assert sse.cpu().tolist() == ref["sse"]
    s, _ = pkg.zonal_sweep(t, 10, 5)
    torch.cuda.synchronize()
    for i, r in enumerate(range(10, 15)):
        assert s[:, i].cpu().tolist() == oc.codec_images(vw, "zonal", r=r)["sse"]
    rec, _, _ = pkg.codec(t, "zonal", r=16)
    torch.cuda.synchronize()
    assert np.max(np.abs(pkg.ssim(t, rec).cpu().numpy() - oq.ssim(vw, rec.cpu().numpy()))) < 1e-9


def test_huge_batch_of_tiny_images():
    """70,000 images of 16x16 (more than a grid's 65,535 y-dimension): forward,
    forward16, the fused codec (zonal, uniform), psnr, the sweep and SSIM."""
    rng = np.random.default_rng(31)
    imgs = rng.integers(0, 256, size=(70000, 16, 16)).astype(np.uint8)
    x = to_dev(imgs)
    Z = oracle_Z(imgs)
    assert np.array_equal(pkg.forward(x).cpu().numpy(), Z)
    rec, sse, _ = pkg.codec(x, "zonal", r=16)
    torch.cuda.synchronize()
    ref = oc.codec_images(imgs, "zonal", r=16)
    assert np.array_equal(rec.cpu().numpy(), ref["recon_img"])
    assert sse.cpu().tolist() == ref["sse"]
    s2 = torch.empty(70000, dtype=torch.int64, device=DEV)
    pkg.dct16a_psnr(x, rec, s2)
    torch.cuda.synchronize()
    assert s2.cpu().tolist() == ref["sse"]
    sw, _ = pkg.zonal_sweep(x, 16, 1)
    torch.cuda.synchronize()
    assert sw[:, 0].cpu().tolist() == ref["sse"]
    ss = pkg.ssim(x, rec).cpu().numpy()
    sel = [0, 65535, 69999]
    assert np.max(np.abs(ss[sel] - np.array(oq.ssim(imgs[sel], rec.cpu().numpy()[sel])))) < 1e-9
    f = (imgs.astype(np.int16) * 4)[:20000]
    fd = to_dev(f)
    rec, sse, _ = pkg.codec(fd, "uniform", step=16)
    torch.cuda.synchronize()
    ref = oc.codec_images(f, "uniform", step=16, bit_depth=10)
    assert sse.cpu().tolist() == ref["sse"]


def test_c_api_demo_runs():
    import subprocess
    import test_abi
    r, out = test_abi._build_c_demo()
    assert r.returncode == 0, r.stderr
    run = subprocess.run([out], capture_output=True, text=True, timeout=120)
    assert run.returncode == 0, run.stdout + run.stderr
    assert "c_api_demo ok" in run.stdout


@pytest.mark.parametrize("mode", [-1, 3, 5])
def test_forward_every_store_mode(mode):
    """Every K1 output path of the product build (DCT16A_OPT_FWD_STORE default,
    3 and 5) is bit-exact, 8- and 10-bit, ragged strips and narrow images."""
    old = pkg.dct16a_get_option(pkg.OPT_FWD_STORE)
    pkg.dct16a_set_option(pkg.OPT_FWD_STORE, mode)
    try:
        for name, imgs in u8_cases():
            if name in ("cfg1", "ragged17x3", "wide", "tiny", "narrow"):
                assert np.array_equal(gpu_Z(to_dev(imgs)), oracle_Z(imgs)), name
        f = synth.frames_10bit([0, 1], H=64, W=272, workers=1)
        assert np.array_equal(gpu_Z(to_dev(f)), oracle_Z(f))
    finally:
        pkg.dct16a_set_option(pkg.OPT_FWD_STORE, old)


@pytest.mark.parametrize("step", [2, 4, 6, 8, 24, 40, 72])
def test_codec_uniform_reconstruction_ties(step, codec_path, uniform_quant):
    """Flat blocks: only the DC level survives, A′ = Δ·q00/16, an exact .5 tie
    whenever Δ·q00 ≡ 8 (mod 16) — the fused kernel must send those pixels to
    the exact decision (round half away from zero)."""
    v = np.arange(256, dtype=np.uint8).reshape(16, 16)
    imgs = np.kron(v, np.ones((16, 16), dtype=np.uint8))[None]          # 256 flat blocks, values 0..255
    _codec_check(imgs, "uniform", 8, step=step)
    f = (np.kron(np.arange(256).reshape(16, 16) * 4 + 1, np.ones((16, 16), dtype=np.int64))).astype(np.int16)[None]
    _codec_check(f, "uniform", 10, step=step)
    ref = oc.codec_images(imgs, "uniform", step=step, bit_depth=8)
    if step in (24, 40, 72):
        assert ref["n_near_ties"] > 0


def _random_case(rng):
    bd = int(rng.choice([8, 10]))
    elem = 1 if bd == 8 else 2
    H = 16 * int(rng.integers(1, 9))
    W = 16 * int(rng.integers(1, 26))
    n = int(rng.integers(1, 4))
    pad_w = 16 * int(rng.integers(0, 3)) // elem          # extra pixels per row (pitch > width)
    pad_h = int(rng.integers(0, 3))                      # extra rows per image (stride > pitch·height)
    hi = 256 if bd == 8 else 1024
    base = rng.integers(0, hi, size=(n, H + pad_h, W + pad_w)).astype(np.uint8 if bd == 8 else np.int16)
    smooth = rng.random() < 0.5
    if smooth:   # AR(1)-like smooth content so that quantisation keeps structure
        field = np.cumsum(np.cumsum(rng.normal(size=base.shape), axis=1), axis=2)
        field = (field - field.min()) / max(1e-9, np.ptp(field)) * (hi - 1)
        base = np.rint(field).astype(base.dtype)
    return bd, base


@pytest.mark.parametrize("seed", range(32))
def test_random_shapes_every_entry(seed):
    """Seeded random geometries (widths 16..400, heights 16..128, pitched and
    strided windows, batches 1-3, 8/10-bit, random r and Δ): forward, the fused
    codec on every kernel, the r-sweep and SSIM against the oracle."""
    rng = np.random.default_rng(1000 + seed)
    bd, base = _random_case(rng)
    n, Hp, Wp = base.shape
    H = max(16, (Hp // 16) * 16)
    W = max(16, (Wp // 16) * 16)
    view = base[:, :H, :W]
    vc = np.ascontiguousarray(view)
    t = to_dev(base)[:, :H, :W]
    assert np.array_equal(gpu_Z(t), oracle_Z(vc))
    r = int(rng.integers(1, 257))
    step = int(rng.integers(1, 100))
    old = pkg.dct16a_get_option(pkg.OPT_CODEC_PATH)
    try:
        for path in (0, 2):
            pkg.dct16a_set_option(pkg.OPT_CODEC_PATH, path)
            for mode in ("zonal", "uniform"):
                rec, sse, _ = pkg.codec(t, mode, r=r, step=step)
                torch.cuda.synchronize()
                ref = oc.codec_images(vc, mode, r=r, step=step, bit_depth=bd)
                assert np.array_equal(rec.cpu().numpy(), ref["recon_img"]), (path, mode, r, step)
                assert sse.cpu().tolist() == ref["sse"], (path, mode)
    finally:
        pkg.dct16a_set_option(pkg.OPT_CODEC_PATH, old)
    r0 = int(rng.integers(1, 250))
    s, _ = pkg.zonal_sweep(t, r0, 3)
    torch.cuda.synchronize()
    for i in range(3):
        assert s[:, i].cpu().tolist() == oc.codec_images(vc, "zonal", r=r0 + i, bit_depth=bd)["sse"]
    rec, _, _ = pkg.codec(t, "zonal", r=r)
    torch.cuda.synchronize()
    got = pkg.ssim(t, rec).cpu().numpy()
    assert np.max(np.abs(got - np.array(oq.ssim(vc, rec.cpu().numpy(), bd)))) < 1e-9


def test_codec_concurrent_streams(codec_path):
    """Eight fused-codec launches in flight on eight streams (zonal r = 32 on
    the band kernel, uniform on the warp kernel; each launch takes its own
    scheduler slot) and 100 launches in a row (slot reuse after reset): every
    reconstruction and SSE vector equals the oracle."""
    imgs = [synth.batch_u8(range(200 + 3 * i, 203 + 3 * i), 64, 384) for i in range(8)]
    xs = [to_dev(a) for a in imgs]
    refs = {m: [oc.codec_images(a, m, r=32, step=16) for a in imgs] for m in ("zonal", "uniform")}
    streams = [torch.cuda.Stream(DEV) for _ in range(8)]
    for mode in ("zonal", "uniform"):
        q = pkg.make_quant(mode, 32, 16)
        recs = [torch.empty_like(x) for x in xs]
        sses = [torch.empty(3, dtype=torch.int64, device=DEV) for _ in xs]
        torch.cuda.synchronize()
        for x, rec, sse, s in zip(xs, recs, sses, streams):
            with torch.cuda.stream(s):
                pkg.dct16a_codec(x, q, sse, rec, None, pkg.desc_of(x), s)
        torch.cuda.synchronize()
        for rec, sse, ref in zip(recs, sses, refs[mode]):
            assert np.array_equal(rec.cpu().numpy(), ref["recon_img"])
            assert sse.cpu().tolist() == ref["sse"]
        for _ in range(100):
            pkg.dct16a_codec(xs[0], q, sses[0], recs[0], None, pkg.desc_of(xs[0]))
        torch.cuda.synchronize()
        assert np.array_equal(recs[0].cpu().numpy(), refs[mode][0]["recon_img"])
        assert sses[0].cpu().tolist() == refs[mode][0]["sse"]


def test_mixed_kernels_concurrent_streams():
    """Different instantiations of the scheduled kernels in flight at once (they
    share one counter array per kernel family): 8-bit int32 forward, 16-bit
    forward, 10-bit forward, zonal codec on bands 3/5/7, uniform codec on 8 and
    10 bits, each on its own stream, three rounds; every result equals the oracle."""
    u8 = synth.batch_u8(range(300, 303), 64, 384)
    u10 = (synth.batch_u8(range(310, 312), 64, 256).astype(np.int16) * 4 + 3).astype(np.int16)
    x8, x10 = to_dev(u8), to_dev(u10)
    z8, z10 = oracle_Z(u8), oracle_Z(u10)
    codec_cases = [(x8, u8, "zonal", 10), (x8, u8, "zonal", 21), (x8, u8, "zonal", 32),
                   (x8, u8, "uniform", 0), (x10, u10, "uniform", 0)]
    refs = [oc.codec_images(a, m, r=max(r, 1), step=16, bit_depth=10 if a.dtype == np.int16 else 8)
            for _, a, m, r in codec_cases]
    streams = [torch.cuda.Stream(DEV) for _ in range(3 + len(codec_cases))]
    for _ in range(3):
        c8 = torch.empty((z8.shape[0], 16, 16), dtype=torch.int32, device=DEV)
        c16 = torch.empty((z8.shape[0], 16, 16), dtype=torch.int16, device=DEV)
        c10 = torch.empty((z10.shape[0], 16, 16), dtype=torch.int32, device=DEV)
        outs = []
        torch.cuda.synchronize()
        with torch.cuda.stream(streams[0]):
            pkg.dct16a_forward(x8, c8, pkg.desc_of(x8), streams[0])
        with torch.cuda.stream(streams[1]):
            pkg.dct16a_forward16(x8, c16, pkg.desc_of(x8), streams[1])
        with torch.cuda.stream(streams[2]):
            pkg.dct16a_forward(x10, c10, pkg.desc_of(x10, 10), streams[2])
        for (x, a, m, r), s in zip(codec_cases, streams[3:]):
            rec = torch.empty_like(x)
            sse = torch.empty(x.shape[0], dtype=torch.int64, device=DEV)
            with torch.cuda.stream(s):
                pkg.dct16a_codec(x, pkg.make_quant(m, max(r, 1), 16), sse, rec, None,
                                 pkg.desc_of(x, 10 if a.dtype == np.int16 else 8), s)
            outs.append((rec, sse))
        torch.cuda.synchronize()
        assert np.array_equal(c8.cpu().numpy(), z8)
        got16 = c16.cpu().numpy().astype(np.int64)
        got16[:, 0, 0] &= 0xFFFF
        assert np.array_equal(got16, z8)
        assert np.array_equal(c10.cpu().numpy(), z10)
        for (rec, sse), ref in zip(outs, refs):
            assert np.array_equal(rec.cpu().numpy(), ref["recon_img"])
            assert sse.cpu().tolist() == ref["sse"]


def test_forward_concurrent_streams():
    """Eight dct16a_forward launches in flight on eight streams (the dynamic
    tile scheduler hands each launch its own counter slot) and 100 launches
    in a row (slot reuse after reset): every result bit-exact."""
    imgs = [synth.batch_u8(range(100 + 4 * i, 104 + 4 * i), 128, 256) for i in range(8)]
    xs = [to_dev(a) for a in imgs]
    outs = [torch.empty((4 * 8 * 16, 16, 16), dtype=torch.int32, device=DEV) for _ in range(8)]
    streams = [torch.cuda.Stream(DEV) for _ in range(8)]
    torch.cuda.synchronize()
    for rep in range(3):
        for x, o, s in zip(xs, outs, streams):
            with torch.cuda.stream(s):
                pkg.dct16a_forward(x, o, pkg.desc_of(x), s)
        torch.cuda.synchronize()
        for a, o in zip(imgs, outs):
            assert np.array_equal(o.cpu().numpy(), oracle_Z(a))
    x, o = xs[0], outs[0]
    for _ in range(100):
        pkg.dct16a_forward(x, o, pkg.desc_of(x))
    torch.cuda.synchronize()
    assert np.array_equal(o.cpu().numpy(), oracle_Z(imgs[0]))


# ------------------------------------------------ scheduler slots, >64 in flight
def test_more_than_64_launches_in_flight_every_family():
    """96 launches of each scheduled kernel family (forward, band codec, warp
    codec) on 96 streams, issued back to back so many are in flight at once:
    the 64 counter slots are reused by launches on other streams, which the
    host orders after the slot's previous launch; every result is exact."""
    nst = 96
    streams = [torch.cuda.Stream(DEV) for _ in range(nst)]
    imgs = [synth.batch_u8([500 + i], 32, 256) for i in range(8)]
    xs = [to_dev(a) for a in imgs]
    zs = [oracle_Z(a) for a in imgs]
    refs = {m: [oc.codec_images(a, m, r=21, step=16) for a in imgs] for m in ("zonal", "uniform")}
    coefs = [torch.full((32, 16, 16), -7, dtype=torch.int32, device=DEV) for _ in range(nst)]
    recs = {m: [torch.zeros_like(xs[0]) for _ in range(nst)] for m in refs}
    sses = {m: [torch.full((1,), -1, dtype=torch.int64, device=DEV) for _ in range(nst)] for m in refs}
    torch.cuda.synchronize()
    for i, s in enumerate(streams):
        x = xs[i % 8]
        with torch.cuda.stream(s):
            pkg.dct16a_forward(x, coefs[i], pkg.desc_of(x), s)
            for m in refs:
                pkg.dct16a_codec(x, pkg.make_quant(m, 21, 16), sses[m][i], recs[m][i], None, pkg.desc_of(x), s)
    torch.cuda.synchronize()
    for i in range(nst):
        assert np.array_equal(coefs[i].cpu().numpy(), zs[i % 8]), i
        for m in refs:
            assert np.array_equal(recs[m][i].cpu().numpy(), refs[m][i % 8]["recon_img"]), (m, i)
            assert sses[m][i].cpu().tolist() == refs[m][i % 8]["sse"], (m, i)


def test_graph_replays_overlap_safely():
    """A launch captured into a CUDA graph takes the static tile schedule (no
    shared counter): replays of one graph overlapping on two streams give the
    exact result, and 130 eager launches afterwards (every slot twice) too."""
    imgs = synth.batch_u8([600, 601], 64, 512)
    x = to_dev(imgs)
    z = oracle_Z(imgs)
    ref = oc.codec_images(imgs, "uniform", step=16)
    coef = torch.zeros((z.shape[0], 16, 16), dtype=torch.int32, device=DEV)
    rec = torch.zeros_like(x)
    sse = torch.zeros(2, dtype=torch.int64, device=DEV)
    q = pkg.make_quant("uniform", 16, 16)
    cs = torch.cuda.Stream(DEV)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=cs):
        pkg.dct16a_forward(x, coef, pkg.desc_of(x), cs)
        pkg.dct16a_codec(x, q, sse, rec, None, pkg.desc_of(x), cs)
    coef.zero_()
    rec.zero_()
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    assert np.array_equal(coef.cpu().numpy(), z)
    assert np.array_equal(rec.cpu().numpy(), ref["recon_img"]) and sse.cpu().tolist() == ref["sse"]
    s1, s2 = torch.cuda.Stream(DEV), torch.cuda.Stream(DEV)
    for _ in range(10):
        with torch.cuda.stream(s1):
            g.replay()
        with torch.cuda.stream(s2):
            g.replay()
    torch.cuda.synchronize()
    assert np.array_equal(coef.cpu().numpy(), z)
    assert np.array_equal(rec.cpu().numpy(), ref["recon_img"])
    for _ in range(130):
        coef.fill_(-1)
        pkg.dct16a_forward(x, coef, pkg.desc_of(x))
        pkg.dct16a_codec(x, q, sse, rec, None, pkg.desc_of(x))
    torch.cuda.synchronize()
    assert np.array_equal(coef.cpu().numpy(), z)
    assert np.array_equal(rec.cpu().numpy(), ref["recon_img"]) and sse.cpu().tolist() == ref["sse"]


# ---------------------------------------- C entries: host pipeline, finaliser
@pytest.mark.parametrize("chunk", [1, 3, 64])
def test_forward_host_c_entry(chunk):
    """dct16a_forward_host: pinned host images -> chunked H2D / forward / D2H on
    two library streams -> pinned host coefficients, bit-exact, for chunk sizes
    that leave a ragged last chunk; 8- and 10-bit, pitched host rows."""
    imgs = synth.batch_u8(range(700, 707), 64, 96)
    h = torch.from_numpy(imgs).pin_memory()
    out = torch.full((7 * 4 * 6, 16, 16), -3, dtype=torch.int32).pin_memory()
    ws = pkg.forward_host(h, out, chunk_images=chunk)
    torch.cuda.current_stream().synchronize()
    assert np.array_equal(out.numpy(), oracle_Z(imgs))
    f = synth.frames_10bit(range(5), H=48, W=80, workers=1)
    wide = np.zeros((5, 48, 96), dtype=np.int16)
    wide[:, :, :80] = f
    hf = torch.from_numpy(wide).pin_memory()[:, :, :80]
    outf = torch.empty((5 * 3 * 5, 16, 16), dtype=torch.int32).pin_memory()
    pkg.forward_host(hf, outf, chunk_images=chunk, workspace=ws)
    torch.cuda.current_stream().synchronize()
    assert np.array_equal(outf.numpy(), oracle_Z(f))


def test_sse_psnr_finaliser():
    """dct16a_sse_psnr: per-item PSNR and the exact total / global PSNR of a
    per-frame SSE vector (config 4's finaliser), against the oracle's formula."""
    rng = np.random.default_rng(5)
    v = rng.integers(0, 2 ** 40, size=1000).astype(np.int64)
    v[7] = 0
    sse = to_dev(v)
    d = pkg.make_desc(3840, 2160, 1, 10)
    psnr, tot, ptot = torch.empty(1000, dtype=torch.float64, device=DEV), torch.empty(1, dtype=torch.int64, device=DEV), torch.empty(1, dtype=torch.float64, device=DEV)
    pkg.dct16a_sse_psnr(sse, 1000, d, psnr, tot, ptot)
    torch.cuda.synchronize()
    P = 3840 * 2160
    assert int(tot.item()) == int(v.sum())
    got = psnr.cpu().tolist()
    for i in range(1000):
        exp = oc.psnr_from_sse(int(v[i]), P, 10)
        assert (math.isinf(exp) and math.isinf(got[i])) or abs(got[i] - exp) < 1e-9
    assert abs(float(ptot.item()) - oc.psnr_from_sse(int(v.sum()), 1000 * P, 10)) < 1e-9
    z = torch.zeros(4, dtype=torch.int64, device=DEV)
    pkg.dct16a_sse_psnr(z, 4, d, None, tot, ptot)
    torch.cuda.synchronize()
    assert int(tot.item()) == 0 and math.isinf(float(ptot.item()))


@pytest.mark.parametrize("world", [2, 3])
def test_config4_sharded_world_gloo_one_gpu(world):
    """The multi-rank config-4 path on this single B200: `world` ranks share
    cuda:0 with a gloo process group over CUDA tensors (NCCL needs one GPU per
    rank); each rank runs the fused codec on its contiguous frame shard, the
    per-frame SSE vector is all-reduced, the library's finaliser gives the
    global PSNR: every frame's SSE and the PSNR equal the oracle's."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={29540 + world}", os.path.join(root, "tools", "run_config4.py"),
           "--frames", "7", "--height", "64", "--width", "208", "--reps", "1", "--dump", "--backend", "gloo"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == world and line["backend"] == "gloo"
    f = synth.frames_10bit(range(7), H=64, W=208, workers=1)
    ref = oc.codec_images(f, "uniform", step=16, bit_depth=10)
    assert line["sse"] == ref["sse"]
    for got, exp in zip(line["psnr"], ref["psnr"]):
        assert abs(got - exp) < 1e-9
    assert abs(line["global_psnr_db"] - oc.psnr_from_sse(sum(ref["sse"]), 7 * 64 * 208, 10)) < 1e-9


@pytest.mark.parametrize("world", [2, 3])
def test_fused_allreduce_ipc_several_processes_one_gpu(world):
    """f2's peer-atomic form across processes: `world` ranks share cuda:0, map
    each other's SSE vectors through CUDA IPC (parallel.IpcSseAllReduce) and
    each rank's kernel adds every one of its frames' SSE into all ranks'
    vectors; every rank's vector equals the gloo all-reduce and the oracle."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={29570 + world}", os.path.join(root, "tools", "run_config4.py"),
           "--frames", "7", "--height", "64", "--width", "208", "--reps", "1", "--dump", "--backend", "gloo", "--ipc"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["ipc_allreduce"] == {"equal_to_collective": True, "n_peers": world}
    ref = oc.codec_images(synth.frames_10bit(range(7), H=64, W=208, workers=1), "uniform", step=16, bit_depth=10)
    assert line["sse"] == ref["sse"]


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="the fused NVLink/NVLS all-reduce needs >= 2 GPUs")
def test_fused_allreduce_multi_gpu_equals_nccl():
    """f2 on >= 2 GPUs: the in-kernel all-reduce (multimem.red on the NVLS
    multicast address when symmetric memory provides one, else peer atomics)
    equals the NCCL all-reduce, frame by frame."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    n = min(torch.cuda.device_count(), 8)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", "--master-port=29551", os.path.join(root, "tools", "run_config4.py"),
           "--frames", "11", "--height", "64", "--width", "208", "--reps", "2", "--dump", "--fused"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["fused_allreduce"]["equal_to_nccl"] is True
    ref = oc.codec_images(synth.frames_10bit(range(11), H=64, W=208, workers=1), "uniform", step=16, bit_depth=10)
    assert line["sse"] == ref["sse"]


@pytest.mark.parametrize("bd", [8, 10])
def test_band_kernel_every_r(bd):
    """The band-pruned zonal kernel (codec path 0) for every r, 1..256 (bands
    3/5/7/11/15; one or two columns per lane; r > 136 on the unpruned band 15),
    8- and 10-bit, on a ragged strip (17 blocks: a partial tile) with pitched
    rows: pixels and SSE equal the oracle, and the warp kernel (path 2) byte
    for byte."""
    hi = 256 if bd == 8 else 1024
    rng = np.random.default_rng(77 + bd)
    if bd == 8:
        base = synth.batch_u8([20, 21], 48, 288)
    else:
        base = synth.frames_10bit([5, 6], H=48, W=288, workers=1)
    base[0, :4, :16] = hi - 1                         # saturated corner: clamping at the top
    base[1, 8:16, 32:64] = 0                          # and at the bottom
    view = base[:, :, :272]
    vc = np.ascontiguousarray(view)
    t = to_dev(base)[:, :, :272]
    old = pkg.dct16a_get_option(pkg.OPT_CODEC_PATH)
    try:
        for r in range(1, 257):
            pkg.dct16a_set_option(pkg.OPT_CODEC_PATH, 0)
            rec, sse, _ = pkg.codec(t, "zonal", r=r)
            pkg.dct16a_set_option(pkg.OPT_CODEC_PATH, 2)
            rec2, sse2, _ = pkg.codec(t, "zonal", r=r)
            torch.cuda.synchronize()
            assert torch.equal(rec, rec2) and torch.equal(sse, sse2), r
            if r in (1, 2, 6, 7, 10, 15, 16, 21, 28, 29, 36, 37, 45, 64, 66, 78, 79, 100, 120, 136, 137, 150, 200, 255, 256):
                ref = oc.codec_images(vc, "zonal", r=r, bit_depth=bd)
                assert np.array_equal(rec.cpu().numpy(), ref["recon_img"]), r
                assert sse.cpu().tolist() == ref["sse"], r
    finally:
        pkg.dct16a_set_option(pkg.OPT_CODEC_PATH, old)
    del rng


def test_fused_allreduce_several_peer_vectors_one_gpu():
    """The n_peers > 1 branch of dct16a_codec_allreduce on one GPU: three
    'ranks' (three frame shards, launched concurrently on three streams) each
    add every frame's SSE into all three per-rank vectors (here plain device
    buffers of one process instead of peer-mapped symmetric memory); every
    vector ends with every frame's SSE, equal to the oracle, and to the NCCL
    form's reduce-by-offset."""
    f = synth.frames_10bit(range(9), H=64, W=208, workers=1)
    x = to_dev(f)
    q = pkg.make_quant("uniform", 16, 16)
    vecs = [torch.zeros(9, dtype=torch.int64, device=DEV) for _ in range(3)]
    peers = [v.data_ptr() for v in vecs]
    streams = [torch.cuda.Stream(DEV) for _ in range(3)]
    torch.cuda.synchronize()
    for rank, (a, b) in enumerate([(0, 3), (3, 5), (5, 9)]):
        shard = x[a:b]
        with torch.cuda.stream(streams[rank]):
            pkg.dct16a_codec_allreduce(shard, q, peers, a, None, pkg.desc_of(shard), streams[rank])
    torch.cuda.synchronize()
    ref = oc.codec_images(f, "uniform", step=16, bit_depth=10)
    for v in vecs:
        assert v.cpu().tolist() == ref["sse"]
