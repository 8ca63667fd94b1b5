"""Pins of the CPU oracle against what the paper and the mathematics fix.

None of these re-types an oracle formula and compares it with itself: each
checks the oracle against a printed value (tests/golden/*, cited), an
independent transcription (factor matrices vs T), a closed form, an
invariant, a brute-force evaluation or a high-precision evaluation.
"""
import decimal
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import synth
from oracle import codec as oc
from oracle import transform as tr

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden_rows(name):
    rows = {}
    for line in open(os.path.join(GOLDEN, name)):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        parts = line.split()
        rows[parts[0]] = parts[1:]
    return rows


def _first_column():
    for line in open(os.path.join(GOLDEN, "t_first_column.txt")):
        if line.strip() and not line.startswith("#"):
            return [int(v) for v in line.split()]


# ------------------------------------------------------------------ T, S
def test_T_entries_and_counts():
    T = tr.build_T()
    assert set(np.unique(T)) <= {-1, 0, 1}
    assert int(np.count_nonzero(T)) == 192
    assert list(np.count_nonzero(T, axis=1)) == [16, 16, 12, 8, 8, 16, 12, 12, 16, 12, 12, 8, 8, 12, 12, 12]
    assert list(T[:, 0]) == _first_column()


def test_T_gram_is_diagonal_and_matches_printed_S():
    T = tr.build_T()
    G = T @ T.T
    assert np.count_nonzero(G - np.diag(np.diag(G))) == 0
    s = tr.build_S_diag()                                      # printed
    assert np.allclose(s * s * np.diag(G), 1.0, rtol=0, atol=1e-15)
    Ch = tr.build_C_hat()
    assert np.max(np.abs(Ch @ Ch.T - np.eye(16))) < 1e-12


# ----------------------------------------------------- Eq. (1) factorisation
def test_factor_product_equals_T():
    assert np.array_equal(tr.factor_product(), tr.build_T())


def test_P2_reading_is_the_unique_row_matching():
    # Reading A1: derive sigma by matching rows of T against M4·M3·M2·P1·M1,
    # independently of the cycle parser, and check uniqueness.
    partial = tr.build_M4() @ tr.build_M3() @ tr.build_M2() @ tr.build_P1() @ tr.build_M1()
    T = tr.build_T()
    sigma = []
    for i in range(16):
        hits = [j for j in range(16) if np.array_equal(partial[j], T[i])]
        assert len(hits) == 1
        sigma.append(hits[0])
    assert sigma == tr.parse_cycles(tr.P2_CYCLES_AS_PRINTED)
    # the other direction of the same cycles must NOT reproduce T
    inv = [0] * 16
    for i, s in enumerate(sigma):
        inv[s] = i
    assert not np.array_equal(tr.build_P2(inv) @ partial, T)


def test_additions_match_table1():
    rows = _golden_rows("table1.txt")
    mult, adds, shifts, total = (int(v) for v in rows["Proposed"])
    c = tr.OpCounter()
    per = {}
    tr.fast_forward_1d(list(range(16)), c, per)
    assert (c.mults, c.adds, c.shifts) == (mult, adds, shifts)
    assert c.adds + c.mults + c.shifts == total == 60
    assert per == {"M1": 16, "P1": 0, "M2": 16, "M3": 24, "M4": 4, "P2": 0}
    # dense T·x: sum over rows of (nonzeros - 1)
    assert int(np.sum(np.count_nonzero(tr.build_T(), axis=1) - 1)) == 176
    ci = tr.OpCounter()
    tr.fast_inverse_1d(list(range(16)), ci)
    assert ci.adds == 60


def test_fast_equals_dense_10000_vectors():
    # hardware co-simulation with 10,000 random 16-point vectors.
    rng = np.random.default_rng(1165)
    T = tr.build_T()
    X = rng.integers(-255, 256, size=(10000, 16))
    for x in X[:2000]:
        assert tr.fast_forward_1d(x) == list(T @ x)
    # vectorised remainder through the stage matrices applied one by one
    Y = X.T.copy()
    for _, F in tr.factor_list():
        Y = F @ Y
    assert np.array_equal(Y, T @ X.T)
    for y in X[:500]:
        assert tr.fast_inverse_1d(y) == list(T.T @ y)


def test_impulse_and_ones():
    col0 = tr.fast_forward_1d([1] + [0] * 15)
    assert col0 == _first_column()
    assert tr.fast_forward_1d([1] * 16) == [16] + [0] * 15


# ------------------------------------------------------------ Table 2
def _tol(printed: str) -> float:
    dec = len(printed.split(".")[1]) if "." in printed else 0
    return 0.5 * 10.0 ** (-dec) + 1e-12


@pytest.mark.parametrize("name,builder", [
    ("Proposed", tr.build_C_hat), ("DCT", tr.build_dct), ("WHT", tr.build_wht_natural)])
def test_table2(name, builder):
    printed = _golden_rows("table2.txt")[name]
    got = tr.table2_row(builder())
    for key, p in zip(["d2", "eps", "mse", "cg", "eta"], printed):
        assert abs(got[key] - float(p)) <= _tol(p), (name, key, got[key], p)


def test_klt_efficiency_is_100():
    assert abs(tr.transform_efficiency(tr.klt()) - 100.0) < 1e-8


def test_dct_rows_orthonormal_and_closed_form_entry():
    C = tr.build_dct()
    assert np.max(np.abs(C @ C.T - np.eye(16))) < 1e-12
    assert abs(C[1, 0] - math.sqrt(2 / 16) * math.cos(math.pi / 32)) < 1e-15
    assert abs(C[1, 0] - 0.351851) < 1e-6


# ------------------------------------------------------------ zig-zag
def test_zigzag_reading_A4():
    z = tr.zigzag()
    assert sorted(z) == [(k, l) for k in range(16) for l in range(16)]
    assert z[:6] == [(0, 0), (0, 1), (1, 0), (2, 0), (1, 1), (0, 2)]
    assert z[-1] == (15, 15)
    d = [k + l for k, l in z]
    assert d == sorted(d)
    assert np.array_equal(tr.zonal_mask(256), np.ones((16, 16), dtype=np.int64))
    with pytest.raises(ValueError):
        tr.zonal_mask(0)
    with pytest.raises(ValueError):
        tr.zonal_mask(257)


# ------------------------------------------------------------- forward
def _rand_blocks(n, maxv, seed):
    return np.random.default_rng(seed).integers(0, maxv + 1, size=(n, 16, 16))


def test_forward_vs_bruteforce_loops():
    X = np.concatenate([_rand_blocks(6, 255, 0), _rand_blocks(2, 1023, 1)])
    Z = oc.forward(X)
    for b in range(len(X)):
        assert np.array_equal(Z[b], oc.forward_bruteforce(X[b]))


def test_forward_properties():
    T = tr.build_T()
    X = _rand_blocks(5000, 255, 2)
    Z = oc.forward(X)
    g = np.diag(T @ T.T)
    W = 2304 // np.outer(g, g)
    # integer Parseval: sum W·Z² = 2304·sum X²
    assert np.array_equal(np.sum(W * Z * Z, axis=(1, 2)), 2304 * np.sum(X * X, axis=(1, 2)))
    # DC = block sum
    assert np.array_equal(Z[:, 0, 0], X.sum(axis=(1, 2)))
    # horizontal mirror -> Z·(-1)^l ; vertical mirror -> Z·(-1)^k ; transpose -> Zᵀ
    sgn = (-1) ** np.arange(16)
    assert np.array_equal(oc.forward(X[:, :, ::-1]), Z * sgn[None, None, :])
    assert np.array_equal(oc.forward(X[:, ::-1, :]), Z * sgn[None, :, None])
    assert np.array_equal(oc.forward(X.transpose(0, 2, 1)), Z.transpose(0, 2, 1))
    # constant block -> DC only; impulse -> outer(T[:, i], T[:, j])
    c = oc.forward(np.full((1, 16, 16), 37))
    assert c[0, 0, 0] == 256 * 37 and np.count_nonzero(c) == 1
    imp = np.zeros((1, 16, 16), dtype=np.int64)
    imp[0, 3, 11] = 1
    assert np.array_equal(oc.forward(imp)[0], np.outer(T[:, 3], T[:, 11]))


def test_forward_integer_ranges_V9():
    T = tr.build_T()
    for maxv, lo, hi, ac in [(255, -32640, 65280, 32640), (1023, -130944, 261888, 130944)]:
        # exact extremes over the pixel box: for each (k, l) the max of
        # sum(sign·x) is maxv·#positive, the min is -maxv·#negative.
        O = np.einsum("ki,lj->klij", T, T)
        pos = (O > 0).sum(axis=(2, 3)) * maxv
        neg = -(O < 0).sum(axis=(2, 3)) * maxv
        assert pos.max() == hi and neg.min() == lo
        pos[0, 0] = 0
        assert max(pos.max(), -neg.min()) == ac
        # the extremes are attained by the sign pattern images
        k, l = np.unravel_index(np.argmax(pos), pos.shape)
        img = np.where(O[k, l] > 0, maxv, 0)[None]
        assert oc.forward(img)[0, k, l] == ac


# ---------------------------------------------------------------- zonal
def test_zonal_r256_is_lossless():
    imgs = synth.batch_u8([0, 1], 64, 64)
    out = oc.codec_images(imgs, "zonal", r=256)
    assert np.array_equal(out["recon_img"], imgs)
    assert out["sse"] == [0, 0] and out["psnr"] == [math.inf, math.inf]
    adv = synth.adversarial_u8()
    assert np.array_equal(oc.codec_images(adv, "zonal", r=256)["recon_img"], adv)


def test_zonal_r1_is_rounded_block_mean():
    X = np.concatenate([_rand_blocks(300, 255, 3), np.full((1, 16, 16), 7)])
    # force an exact .5 tie: block sum = 128·(2·40+1) -> mean 40.5 -> 41
    tie = np.full((1, 16, 16), 40)
    tie[0, :8, :] = 41
    X = np.concatenate([X, tie])
    rec = oc.zonal_codec(X, 1)["recon"]
    s = X.sum(axis=(1, 2))
    want = np.floor(s / 256 + 0.5).astype(np.int64)          # mean >= 0: half-up == half-away
    assert np.array_equal(rec, np.broadcast_to(want[:, None, None], rec.shape))
    assert rec[-1, 0, 0] == 41


@pytest.mark.parametrize("r", [1, 2, 15, 16, 17, 32, 64, 128, 255])
def test_zonal_exact_numerator_equals_float_definition(r):
    X = _rand_blocks(400, 255, r)
    out = oc.zonal_codec(X, r)
    Af = oc.zonal_recon_float(X, r)               # Ĉᵀ·B′·Ĉ with the printed S
    assert np.max(np.abs(Af - out["N"] / 2304.0)) < 1e-9
    # scaled stage: B′ = S·Z·S ⊙ M with S printed
    s = tr.build_S_diag()
    assert np.allclose(out["scaled"], np.outer(s, s) * out["Zm"], rtol=1e-13, atol=1e-12)


def test_zonal_numerator_against_fractions():
    T = tr.build_T()
    g = [int(v) for v in np.diag(T @ T.T)]
    X = _rand_blocks(2, 255, 11)
    for r in (16, 32):
        out = oc.zonal_codec(X, r)
        M = tr.zonal_mask(r)
        for b in range(2):
            Zm = out["Zm"][b]
            for i in (0, 5, 15):
                for j in (0, 7, 14):
                    a = Fraction(0)
                    for k in range(16):
                        for l in range(16):
                            if M[k, l]:
                                # Ĉᵀ·(S·Z·S ⊙ M)·Ĉ with S² = 1/g exactly
                                a += Fraction(int(Zm[k, l]) * int(T[k, i]) * int(T[l, j]), g[k] * g[l])
                    assert a == Fraction(int(out["N"][b, i, j]), 2304)
                    want = math.floor(abs(a) + Fraction(1, 2)) * (1 if a >= 0 else -1)
                    assert out["recon"][b, i, j] == min(255, max(0, want))


def test_zonal_rounding_ties_need_exact_decision_V11():
    # on the config-1 image, exact .5 ties occur (V11): the oracle decides them
    # on the integer numerator and rounds them away from zero.
    img = synth.image_u8(0)[None]
    X = oc.to_blocks(img.astype(np.int64))
    out = oc.zonal_codec(X, 16)
    ties = (out["N"] % 2304) == 1152
    assert ties.sum() > 0
    rec_expect = np.clip((out["N"][ties] + 1152) // 2304, 0, 255)
    assert np.array_equal(out["recon"][ties], rec_expect)


def test_psnr_sanity_config1_V14():
    img = synth.image_u8(0)[None]
    p = oc.codec_images(img, "zonal", r=16)["psnr"][0]
    d = oc.dct_zonal_images(img, 16)["psnr"][0]
    assert 20.0 < p < d < 35.0                 # approx below exact DCT at r=16
    assert abs(oc.ape(p, d) - 5.4) < 1.0       # ~5% (paper's Lena: 4.97%)
    p1 = oc.codec_images(img, "zonal", r=1)["psnr"][0]
    assert p1 == oc.dct_zonal_images(img, 1)["psnr"][0]     # DC rows identical


# -------------------------------------------------------------- uniform
def test_uniform_q_matches_decimal():
    rng = np.random.default_rng(5)
    Z = rng.integers(-261888, 261889, size=(40, 16, 16))
    Z[:, 0, 0] = rng.integers(0, 261889, size=40)
    for step in (1, 3, 16, 40):
        q = oc.uniform_q(Z, step)
        for _ in range(500):
            b, k, l = rng.integers(0, 40), rng.integers(0, 16), rng.integers(0, 16)
            assert q[b, k, l] == oc.uniform_q_decimal(int(Z[b, k, l]), k, l, step)


def test_uniform_q_forced_ties_round_away():
    T = tr.build_T()
    g = np.diag(T @ T.T)
    step = 16
    for k in range(16):
        for l in range(16):
            G = int(g[k] * g[l])
            r = math.isqrt(G)
            if r * r != G:
                continue                        # irrational cell: no exact tie
            for m in (0, 1, 5, 37):
                # |B|/Δ = m + 1/2 exactly  <=>  Z = (2m+1)·Δ·sqrt(G)/2
                z = (2 * m + 1) * step * r // 2
                assert (2 * m + 1) * step * r % 2 == 0
                Z = np.zeros((1, 16, 16), dtype=np.int64)
                Z[0, k, l] = z
                assert oc.uniform_q(Z, step)[0, k, l] == m + 1
                Z[0, k, l] = -z
                assert oc.uniform_q(Z, step)[0, k, l] == -(m + 1)
                Z[0, k, l] = z - 1
                assert oc.uniform_q(Z, step)[0, k, l] == m


def test_uniform_psnr_decreases_with_step():
    f = synth.frame_10bit(0, H=128, W=256)[None]
    ps = [oc.codec_images(f, "uniform", step=s, bit_depth=10)["psnr"][0] for s in (1, 4, 16, 64)]
    assert ps[0] > ps[1] > ps[2] > ps[3]
    assert ps[0] > 55.0                          # Δ=1: near-lossless (B irrational, not lossless)
    assert 43.0 < ps[2] < 50.0                   # Δ=16 on cfg4-like data ≈ 46.9 dB (V12)


def test_uniform_recon_pixel_against_decimal():
    f = synth.frame_10bit(1, H=32, W=64)[None]
    out = oc.codec_images(f, "uniform", step=16, bit_depth=10)
    q = out["q"]
    rng = np.random.default_rng(9)
    for _ in range(40):
        by, bx, i, j = rng.integers(0, 2), rng.integers(0, 4), rng.integers(0, 16), rng.integers(0, 16)
        d = oc._uniform_pixel_decimal(q[0, by, bx], i, j, 16)
        want = int(d.to_integral_value(rounding=decimal.ROUND_HALF_UP))
        assert out["recon"][0, by, bx, i, j] == min(1023, max(0, want))


# ----------------------------------------------------------------- PSNR
def test_psnr_closed_forms():
    a = np.zeros((1, 16, 16), dtype=np.int64)
    b = a + 1
    s = oc.sse(a, b)[0]
    assert abs(oc.psnr_from_sse(s, 256, 8) - 48.1308) < 1e-4       # 10·log10(65025)
    w = a + 255
    assert abs(oc.psnr_from_sse(oc.sse(a, w)[0], 256, 8)) < 1e-12  # black vs white
    assert oc.psnr_from_sse(0, 256, 8) == math.inf
    # valid_height: errors in padding rows are ignored
    c = a.copy()
    c[0, 12:, :] = 9
    assert oc.sse(a, c, valid_height=12) == [0]


# ------------------------------------- uniform reconstruction, exact decisions
def _fraction_recon(qb, step):
    """A′ = Σ_kl T_ki·T_lj·Δ·q_kl/sqrt(g_k g_l) with Fractions, valid when every
    non-zero q_kl sits in a rational cell (g_k g_l a perfect square)."""
    T = tr.build_T()
    g = np.diag(T @ T.T)
    A = [[Fraction(0)] * 16 for _ in range(16)]
    for k in range(16):
        for l in range(16):
            if qb[k][l] == 0:
                continue
            G = int(g[k] * g[l])
            r = math.isqrt(G)
            assert r * r == G
            c = Fraction(step * int(qb[k][l]), r)
            for i in range(16):
                for j in range(16):
                    A[i][j] += c * int(T[k, i]) * int(T[l, j])
    return A


def _round_half_away_fraction(v):
    m = math.floor(abs(v) + Fraction(1, 2))
    return m if v >= 0 else -m


def test_uniform_components_equal_float_definition():
    """144·A′/Δ = Σ_d sqrt(d)·J_d (exact components) against the float64 dense
    definition Ĉᵀ·(Δq)·Ĉ on random levels."""
    rng = np.random.default_rng(21)
    q = rng.integers(-300, 301, size=(20, 16, 16))
    for step in (1, 7, 16):
        J = oc.uniform_recon_components(q)
        val = sum(math.sqrt(d) * J[d].astype(np.float64) for d in oc.SQRT_BASIS) * step / 144.0
        assert np.max(np.abs(val - oc.uniform_recon_float(q, step))) < 1e-9


@pytest.mark.parametrize("case", ["flat_dc", "bb_cell", "random_rational"])
def test_uniform_recon_exact_ties_rational_cells(case):
    """Exact .5 ties of the reconstruction (possible only when the irrational
    parts cancel) round away from zero: checked against Fractions."""
    T = tr.build_T()
    g = np.diag(T @ T.T)
    rational = np.array([[math.isqrt(int(g[k] * g[l])) ** 2 == g[k] * g[l] for l in range(16)] for k in range(16)])
    if case == "flat_dc":           # Δ=24, q00=1: A′ = 24/16 = 1.5 everywhere -> 2
        step, qb = 24, np.zeros((1, 16, 16), dtype=np.int64)
        qb[0, 0, 0] = 1
    elif case == "bb_cell":         # Δ=6, q00=8, q22=1: A′ = 3 ± 1/2 at T_2i·T_2j = ±1
        step, qb = 6, np.zeros((1, 16, 16), dtype=np.int64)
        qb[0, 0, 0], qb[0, 2, 2] = 8, 1
    else:
        step = 6
        rng = np.random.default_rng(4)
        qb = rng.integers(-3, 4, size=(6, 16, 16)) * rational
        qb[:, 0, 0] = rng.integers(20, 60, size=6)
    out = oc.uniform_inverse_levels(qb, step, bit_depth=10)
    n_ties = 0
    for b in range(qb.shape[0]):
        A = _fraction_recon(qb[b], step)
        for i in range(16):
            for j in range(16):
                n_ties += (A[i][j] - math.floor(A[i][j])) == Fraction(1, 2)
                want = min(1023, max(0, _round_half_away_fraction(A[i][j])))
                assert out["recon"][b, i, j] == want, (b, i, j, A[i][j])
    assert n_ties > 0
    if case != "flat_dc":
        assert out["n_near_ties"] > 0


def test_uniform_recon_near_ties_irrational_vs_decimal():
    """Pixels whose float64 value lies within 1e-3 of a .5 boundary, with
    irrational parts, against a 80-digit evaluation of the dense definition."""
    rng = np.random.default_rng(13)
    q = rng.integers(-2, 3, size=(400, 16, 16))
    q[:, 0, 0] = rng.integers(30, 90, size=400)
    step = 16
    out = oc.uniform_inverse_levels(q, step, bit_depth=10)
    A = out["A"]
    frac = np.abs(A) - np.floor(np.abs(A))
    idx = np.argwhere(np.abs(frac - 0.5) < 1e-3)
    assert len(idx) >= 5
    for b, i, j in idx[:40]:
        d = oc._uniform_pixel_decimal(q[b], int(i), int(j), step, prec=80)
        want = int(d.to_integral_value(rounding=decimal.ROUND_HALF_UP))
        assert out["recon"][b, i, j] == min(1023, max(0, want))


# ------------------------------------------------------------------ SSIM
from oracle import quality as oq  # noqa: E402


def test_ssim_identity_negative_and_window():
    img = synth.image_u8(3, 48, 64)
    assert oq.ssim(img[None], img[None])[0] == pytest.approx(1.0, abs=1e-12)
    assert oq.ssim(img[None], (255 - img)[None])[0] < 0.5
    w = oq.gaussian_window()
    assert abs(w.sum() - 1.0) < 1e-15 and w.shape == (11, 11) and np.allclose(w, w.T)
    assert np.argmax(w) == 60                       # centre tap (5, 5)


def test_ssim_constant_images_closed_form():
    # constant a vs constant b: σ = 0, so SSIM = (2ab + C1)/(a² + b² + C1) (Wang 2004 eq. 13)
    C1 = (0.01 * 255) ** 2
    for a, b in [(10, 200), (128, 129), (0, 255)]:
        x = np.full((1, 16, 16), a, dtype=np.uint8)
        y = np.full((1, 16, 16), b, dtype=np.uint8)
        want = (2 * a * b + C1) / (a * a + b * b + C1)
        assert oq.ssim(x, y)[0] == pytest.approx(want, abs=1e-12)


def test_ssim_against_straight_line_loops():
    rng = np.random.default_rng(8)
    x = synth.image_u8(4, 16, 24)
    y = np.clip(x.astype(int) + rng.integers(-20, 21, size=x.shape), 0, 255).astype(np.uint8)
    assert oq.ssim(x[None], y[None])[0] == pytest.approx(oq.ssim_bruteforce(x, y), abs=1e-12)
    f = synth.frame_10bit(3, H=16, W=16)
    g = np.clip(f.astype(int) + 7, 0, 1023)
    assert oq.ssim(f[None], g[None], bit_depth=10)[0] == pytest.approx(oq.ssim_bruteforce(f, g, 10), abs=1e-12)


# ------------------------------------------------- whole-image block tiling
# Pins of oracle.codec.to_blocks / from_blocks themselves (PAPER.md:866-869:
# the image is split into disjoint 16x16 blocks A_k; reading A3: all blocks,
# row-major; reading A5: Z = T·X·Tᵀ with X's first index the image row).
# These go through whole images, so an in-block transpose or a swapped block
# order inside the tiler fails them.

def test_to_blocks_matches_pixel_loops():
    rng = np.random.default_rng(21)
    imgs = rng.integers(0, 256, size=(2, 48, 80))          # 3 x 5 blocks, non-square
    Xb = oc.to_blocks(imgs)
    assert Xb.shape == (2, 3, 5, 16, 16)
    for n in range(2):
        for by in range(3):
            for bx in range(5):
                for i in range(16):
                    for j in range(16):
                        assert Xb[n, by, bx, i, j] == imgs[n, 16 * by + i, 16 * bx + j]
    assert np.array_equal(oc.from_blocks(Xb), imgs)
    # from_blocks on its own: block (by, bx) entry (i, j) lands at pixel (16by+i, 16bx+j)
    blk = np.arange(2 * 3 * 5 * 256).reshape(2, 3, 5, 16, 16)
    img = oc.from_blocks(blk)
    for n, by, bx, i, j in [(0, 0, 0, 0, 1), (1, 2, 4, 15, 0), (0, 1, 3, 2, 9), (1, 0, 2, 7, 15)]:
        assert img[n, 16 * by + i, 16 * bx + j] == blk[n, by, bx, i, j]


def test_whole_image_horizontal_ramp_has_energy_in_row_zero_only():
    # X[i][j] = j + c_b inside block b: X = 1·(j + c_b)ᵀ, so Z = (T·1)(T·(j+c_b))ᵀ.
    # T·1 = 16·e₀ (row 0 of T is all ones; every other row is
    # orthogonal to it), hence only the row k = 0 (vertical frequency 0) of Z
    # is non-zero, and Z[0][0] = 16·(120 + 16·c_b) with c_b = by·BX + bx.
    BY, BX = 3, 4
    img = np.zeros((1, 16 * BY, 16 * BX), dtype=np.int64)
    for by in range(BY):
        for bx in range(BX):
            img[0, 16 * by:16 * by + 16, 16 * bx:16 * bx + 16] = np.arange(16)[None, :] + (by * BX + bx)
    Z = oc.forward(oc.to_blocks(img))
    assert np.count_nonzero(Z[..., 1:, :]) == 0
    assert np.count_nonzero(Z[..., 0, 1:]) > 0
    c = np.arange(BY * BX).reshape(BY, BX)
    assert np.array_equal(Z[0, :, :, 0, 0], 16 * (120 + 16 * c))
    # the vertical ramp puts its energy in column l = 0 only
    Zv = oc.forward(oc.to_blocks(img.transpose(0, 2, 1).copy()))
    assert np.count_nonzero(Zv[..., :, 1:]) == 0


def test_whole_image_in_block_mirrors():
    # Mirroring every block left-right inside the image gives Z·(-1)^l and
    # top-bottom gives Z·(-1)^k: T[l][15-j] = (-1)^l·T[l][j] (even/odd rows of
    # T) with l the horizontal frequency (reading A5).
    imgs = synth.image_u8(5, 64, 96)[None].astype(np.int64)
    mir_h = imgs.reshape(1, 4, 16, 6, 16)[:, :, :, :, ::-1].reshape(imgs.shape)
    mir_v = imgs.reshape(1, 4, 16, 6, 16)[:, :, ::-1, :, :].reshape(imgs.shape)
    Z = oc.forward(oc.to_blocks(imgs))
    sgn = (-1) ** np.arange(16)
    assert np.array_equal(oc.forward(oc.to_blocks(mir_h)), Z * sgn[None, None, None, None, :])
    assert np.array_equal(oc.forward(oc.to_blocks(mir_v)), Z * sgn[None, None, None, :, None])
    # and the two are distinguishable on this input (odd k and odd l both present)
    assert np.any(Z[..., 1::2, :] != 0) and np.any(Z[..., :, 1::2] != 0)
    assert not np.array_equal(Z * sgn[None, None, None, None, :], Z * sgn[None, None, None, :, None])


def test_codec_images_keeps_horizontal_detail_in_first_row():
    # The zonal pipeline through the tiler: a per-block horizontal ramp keeps
    # only (0, l) coefficients, and zig-zag r = 3 keeps (0,0),(0,1),(1,0)
    # (reading A4), so the reconstruction depends on j only inside each block.
    img = np.tile(np.arange(16, dtype=np.int64) * 8 + 40, (1, 32, 2))
    rec = oc.codec_images(img, "zonal", r=3)["recon_img"]
    assert np.all(rec == rec[:, :1, :])                        # constant down each column
    assert rec[0, 0, 0] < rec[0, 0, 15]                        # the ramp survives along j


# -------------------------------------------------------- SSIM window sigma
def test_ssim_window_is_gaussian_sigma_1p5():
    # Wang et al. 2004 (the source PAPER.md:911-917 cites; reading A21): an
    # 11x11 circular-symmetric Gaussian with standard deviation 1.5 samples,
    # normalised to unit sum.  Check the taps against the library Gaussian
    # filter (scipy.ndimage, sigma = 1.5, radius 5) applied to an impulse.
    from scipy import ndimage
    imp = np.zeros((11, 11))
    imp[5, 5] = 1.0
    ref = ndimage.gaussian_filter(imp, sigma=1.5, truncate=5 / 1.5, mode="constant")
    assert np.max(np.abs(oq.gaussian_window() - ref)) < 1e-15
    w = oq.gaussian_window()
    # neighbour / centre tap = exp(-1/(2·1.5²)) = exp(-1/4.5) = 0.80073740...
    assert w[5, 6] / w[5, 5] == pytest.approx(0.8007374029168081, rel=1e-14)
    assert w[0, 0] / w[5, 5] == pytest.approx(math.exp(-50 / 4.5), rel=1e-12)


def test_ssim_against_library_gaussian_filter():
    # An independent SSIM: local moments from scipy.ndimage.gaussian_filter
    # (sigma 1.5, 11 taps), cropped to the fully contained windows.
    from scipy import ndimage
    rng = np.random.default_rng(31)
    x = synth.image_u8(6, 40, 56).astype(np.float64)
    y = np.clip(x + rng.integers(-25, 26, size=x.shape), 0, 255)
    f = lambda a: ndimage.gaussian_filter(a, sigma=1.5, truncate=5 / 1.5, mode="constant")[5:-5, 5:-5]
    C1, C2 = (0.01 * 255) ** 2, (0.03 * 255) ** 2
    mx, my = f(x), f(y)
    vx, vy, cxy = f(x * x) - mx * mx, f(y * y) - my * my, f(x * y) - mx * my
    m = ((2 * mx * my + C1) * (2 * cxy + C2)) / ((mx * mx + my * my + C1) * (vx + vy + C2))
    assert oq.ssim(x.astype(np.uint8)[None], y.astype(np.uint8)[None])[0] == pytest.approx(m.mean(), abs=1e-12)
