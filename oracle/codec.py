"""Oracle, part 2: the §4 block-compression pipeline of arXiv 1606.05562 —
disjoint 16x16 blocks, 2-D transform, zig-zag zonal (or uniform) quantisation
with S absorbed, inverse, reconstruction and PSNR.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Dense matrix products in
float64 on integer-valued data (exact: every partial sum is an integer far
below 2^53) or exact Python integers; no blocking, fusion or butterflies.
"""
from __future__ import annotations

import decimal
import math

import numpy as np

from . import transform as tr

B = 16
T = tr.build_T()
T_F = T.astype(np.float64)
G = tr.gram_diag(T)                         # g = diag(T·Tᵀ)
C_HAT = tr.build_C_hat()                    # Ĉ = S·T
GG = np.outer(G, G)                         # g_k·g_l
W_INT = 2304 // GG                          # 2304/(g_k g_l) ∈ {9,12,16,18,24,36}
assert np.all(W_INT * GG == 2304)


# ----------------------------------------------------------------- blocks
def to_blocks(imgs: np.ndarray) -> np.ndarray:
    """(n, H, W) -> (n, H/16, W/16, 16, 16): disjoint 16x16 blocks A_k in
    row-major block order (reading A3: all blocks)."""
    n, H, W = imgs.shape
    if H % B or W % B:
        raise ValueError("image dims must be multiples of 16")
    x = imgs.reshape(n, H // B, B, W // B, B)
    return x.transpose(0, 1, 3, 2, 4).copy()


def from_blocks(blocks: np.ndarray) -> np.ndarray:
    """Inverse of to_blocks: reassemble (n, BY, BX, 16, 16) into (n, H, W)."""
    n, BY, BX, _, _ = blocks.shape
    return blocks.transpose(0, 1, 3, 2, 4).reshape(n, BY * B, BX * B).copy()


def _integral(a: np.ndarray) -> np.ndarray:
    r = np.rint(a)
    assert np.array_equal(r, a), "expected an exactly integral float64 product"
    return r.astype(np.int64)


# ---------------------------------------------------------------- forward
def forward(X: np.ndarray) -> np.ndarray:
    """Z = T·X·Tᵀ per block (PAPER.md:870-880 with C̃ replaced by T, whose
    scale S is absorbed into quantisation; reading A5 for
    orientation: k = row = vertical frequency).  int64 out."""
    Xf = X.astype(np.float64)
    return _integral(T_F @ Xf @ T_F.T)


def forward_bruteforce(X16: np.ndarray) -> np.ndarray:
    """Z[k][l] = sum_i sum_j T[k][i]·X[i][j]·T[l][j] with Python integers, one
    16x16 block; the loop form of the same definition (small-case pin)."""
    Z = [[0] * B for _ in range(B)]
    for k in range(B):
        for l in range(B):
            s = 0
            for i in range(B):
                if T[k, i] == 0:
                    continue
                for j in range(B):
                    s += int(T[k, i]) * int(X16[i][j]) * int(T[l, j])
            Z[k][l] = s
    return np.array(Z, dtype=np.int64)


# ------------------------------------------------------- zonal (§4, r kept)
def zonal_stage(Z: np.ndarray, r: int) -> np.ndarray:
    """Z ⊙ M_r — keep the first r zig-zag coefficients."""
    return Z * tr.zonal_mask(r)


def scaled_2d(X: np.ndarray) -> np.ndarray:
    """B = Ĉ·X·Ĉᵀ, float64 dense products."""
    return C_HAT @ X.astype(np.float64) @ C_HAT.T


def zonal_scaled(X: np.ndarray, r: int) -> np.ndarray:
    """B′ = (Ĉ·X·Ĉᵀ) ⊙ M_r, PAPER.md:874-894 (float64)."""
    return scaled_2d(X) * tr.zonal_mask(r)


def zonal_recon_float(X: np.ndarray, r: int) -> np.ndarray:
    """A′ = Ĉᵀ·B′·Ĉ, PAPER.md:896-901 (float64, the paper's definition)."""
    return C_HAT.T @ zonal_scaled(X, r) @ C_HAT


def zonal_numerator(Zm: np.ndarray) -> np.ndarray:
    """N = Tᵀ·(W ⊙ Zm)·T with W = 2304/(g_k g_l): since Ĉ = S·T and S² = 1/g,
    Ĉᵀ·(S·Z·S ⊙ M)·Ĉ = Tᵀ·(Z ⊙ M / (g_k g_l))·T = N / 2304 exactly
    (PAPER.md:309-344 with 896-901).  Exact int64."""
    return _integral(T_F.T @ (W_INT * Zm).astype(np.float64) @ T_F)


def round_half_away_rational(N: np.ndarray, den: int) -> np.ndarray:
    """round-half-away-from-zero of N/den for integer N (reading A6)."""
    N = np.asarray(N, dtype=np.int64)
    mag = (np.abs(N) + den // 2) // den            # den even: ties go up in magnitude
    return np.sign(N) * mag


def clamp_pixels(v: np.ndarray, bit_depth: int) -> np.ndarray:
    """clamp to [0, 2^b - 1] (reading A6)."""
    return np.clip(v, 0, (1 << bit_depth) - 1)


def zonal_codec(X: np.ndarray, r: int, bit_depth: int = 8) -> dict:
    """The §4 pipeline for a stack of blocks X (..., 16, 16) with zonal r.

    Returns Z, Zm (= Z ⊙ M_r, the integer quantised stage), scaled (= B′,
    float64), N (exact reconstruction numerator) and recon (pixels, rounding
    decided on the exact rational N/2304 — reading A6, V11)."""
    Z = forward(X)
    Zm = zonal_stage(Z, r)
    N = zonal_numerator(Zm)
    recon = clamp_pixels(round_half_away_rational(N, 2304), bit_depth)
    return {"Z": Z, "Zm": Zm, "scaled": zonal_scaled(X, r), "N": N, "recon": recon}


# --------------------------------------------- uniform (reading A9, A10)
def isqrt_array(n: np.ndarray) -> np.ndarray:
    """floor(sqrt(n)) for non-negative int64 n, exact (float estimate then
    integer correction until r² <= n < (r+1)²)."""
    n = np.asarray(n, dtype=np.int64)
    r = np.floor(np.sqrt(n.astype(np.float64))).astype(np.int64)
    for _ in range(4):
        hi = r * r > n
        r = np.where(hi, r - 1, r)
        lo = (r + 1) * (r + 1) <= n
        r = np.where(lo, r + 1, r)
    assert np.all(r * r <= n) and np.all((r + 1) * (r + 1) > n)
    return r


def uniform_q(Z: np.ndarray, step: int) -> np.ndarray:
    """q = sign(B)·floor(|B|/Δ + 1/2) on B = Ĉ·X·Ĉᵀ = Z/sqrt(g_k g_l)
    (reading A9), decided exactly: m is the largest integer with
    (2m-1)·Δ·sqrt(G) <= 2|Z|, i.e. m = (isqrt(floor(4Z²/(Δ²G))) + 1) // 2."""
    Z = np.asarray(Z, dtype=np.int64)
    Gb = np.broadcast_to(GG, Z.shape)
    t = (4 * Z * Z) // (step * step * Gb)
    m = (isqrt_array(t) + 1) // 2
    return np.sign(Z) * m


def uniform_q_decimal(z: int, k: int, l: int, step: int, prec: int = 50) -> int:
    """One coefficient of uniform_q evaluated with `decimal` at `prec` digits
    (independent check of the exact integer decision)."""
    ctx = decimal.Context(prec=prec)
    b = ctx.divide(decimal.Decimal(abs(z)), ctx.sqrt(decimal.Decimal(int(G[k] * G[l]))))
    v = ctx.add(ctx.divide(b, decimal.Decimal(step)), decimal.Decimal("0.5"))
    m = int(v.to_integral_value(rounding=decimal.ROUND_FLOOR))
    return m if z >= 0 else -m


def uniform_recon_float(q: np.ndarray, step: int) -> np.ndarray:
    """A′ = Ĉᵀ·(Δ·q)·Ĉ (PAPER.md:896-901 with B′ = Δq), float64."""
    return C_HAT.T @ (step * q).astype(np.float64) @ C_HAT


def _uniform_pixel_decimal(qb: np.ndarray, i: int, j: int, step: int, prec: int = 50) -> decimal.Decimal:
    """A′[i][j] = Σ_kl T_ki·T_lj·Δ·q_kl/sqrt(g_k g_l) evaluated term by term
    with `decimal` at `prec` digits (an independent check of the inverse)."""
    ctx = decimal.Context(prec=prec)
    acc = decimal.Decimal(0)
    for k in range(B):
        for l in range(B):
            if qb[k, l] == 0 or T[k, i] == 0 or T[l, j] == 0:
                continue
            num = decimal.Decimal(int(step * qb[k, l] * T[k, i] * T[l, j]))
            acc = ctx.add(acc, ctx.divide(num, ctx.sqrt(decimal.Decimal(int(G[k] * G[l])))))
    return acc


def round_half_away_float(a: np.ndarray) -> np.ndarray:
    return np.sign(a) * np.floor(np.abs(a) + 0.5)


# Exact form of the uniform reconstruction (reading A10).  Each weight
# 144·s_k·s_l = 144/sqrt(G), G = g_k·g_l (S of PAPER.md:315-329), is written as
# an integer times sqrt(d) with d square-free: sqrt(G) = a·sqrt(d) gives
# 144/sqrt(G) = (144/(a·d))·sqrt(d).  Then
#     144·A′/Δ = Σ_d sqrt(d) · J_d,   J_d = Tᵀ·(K_d ⊙ q)·T   (exact integers),
# with K_d[k][l] = 144/(a·d) where the cell's square-free part is d, else 0.
def _squarefree_split(G: int) -> tuple[int, int]:
    """sqrt(G) = a·sqrt(d), d square-free (G > 0)."""
    a, d = 1, G
    f = 2
    while f * f <= d:
        while d % (f * f) == 0:
            d //= f * f
            a *= f
        f += 1
    return a, d


SQRT_BASIS = (1, 2, 3, 6)


def _basis_weights() -> dict:
    K = {d: np.zeros((B, B), dtype=np.int64) for d in SQRT_BASIS}
    for k in range(B):
        for l in range(B):
            a, d = _squarefree_split(int(GG[k, l]))
            assert 144 % (a * d) == 0
            K[d][k, l] = 144 // (a * d)
    return K


K_BASIS = _basis_weights()


def uniform_recon_components(q: np.ndarray) -> dict:
    """J_d = Tᵀ·(K_d ⊙ q)·T for d in (1, 2, 3, 6): 144·A′/Δ = Σ_d sqrt(d)·J_d
    exactly (int64; dense products of PAPER.md:896-901 with Ĉ = S·T)."""
    return {d: _integral(T_F.T @ (K_BASIS[d] * q).astype(np.float64) @ T_F) for d in SQRT_BASIS}


def round_half_away_exact_uniform(J: dict, step: int, idx: tuple) -> int:
    """round_half_away(A′) for one pixel from its exact components (reading
    A6/A10).  If the irrational parts vanish the value is the rational
    Δ·J_1/144 and is rounded exactly (ties away from zero).  Otherwise A′ is
    irrational, so it is not a tie, and a 60-digit evaluation decides; the
    distance of such a value to a half-integer is bounded below by the norm of
    a non-zero algebraic integer of Q(√2, √3) over its conjugates (> 1e-40
    here), far above the 1e-55 evaluation error."""
    j = {d: int(J[d][idx]) for d in SQRT_BASIS}
    if j[2] == 0 and j[3] == 0 and j[6] == 0:
        return int(round_half_away_rational(np.array([step * j[1]]), 144)[0])
    ctx = decimal.Context(prec=60)
    v = decimal.Decimal(0)
    for d in SQRT_BASIS:
        v = ctx.add(v, ctx.multiply(decimal.Decimal(j[d]), ctx.sqrt(decimal.Decimal(d))))
    v = ctx.divide(ctx.multiply(v, decimal.Decimal(step)), decimal.Decimal(144))
    frac = abs(v) - abs(v).to_integral_value(rounding=decimal.ROUND_FLOOR)
    assert abs(frac - decimal.Decimal("0.5")) > decimal.Decimal("1e-40")
    return int(v.to_integral_value(rounding=decimal.ROUND_HALF_UP))


def uniform_codec(X: np.ndarray, step: int, bit_depth: int = 10) -> dict:
    """Forward, exact uniform q, then the inverse stage of uniform_inverse_levels
    (float64 reconstruction, reading A10, exact decisions near ties)."""
    Z = forward(X)
    q = uniform_q(Z, step)
    inv = uniform_inverse_levels(q, step, bit_depth)
    return {"Z": Z, "q": q, "scaled": scaled_2d(X), "recon": inv["recon"], "n_near_ties": inv["n_near_ties"]}


def uniform_inverse_levels(q: np.ndarray, step: int, bit_depth: int = 10) -> dict:
    """The inverse stage on levels q (..., 16, 16): A′ = Ĉᵀ·(Δq)·Ĉ in float64
    (PAPER.md:896-901), round half away and clamp (reading A6).  Any pixel
    within 1e-9 of a .5 boundary (the float64 dense product errs by < 1e-11)
    is decided exactly from its components J_d (round_half_away_exact_uniform)."""
    q = np.asarray(q, dtype=np.int64)
    A = uniform_recon_float(q, step)
    frac = np.abs(A) - np.floor(np.abs(A))
    near = np.argwhere(np.abs(frac - 0.5) < 1e-9)
    rec = round_half_away_float(A)
    if len(near):
        J = uniform_recon_components(q)
        for idx in near:
            rec[tuple(int(v) for v in idx)] = round_half_away_exact_uniform(J, step, tuple(int(v) for v in idx))
    return {"A": A, "recon": clamp_pixels(rec.astype(np.int64), bit_depth), "n_near_ties": len(near)}


# ------------------------------------------------------- SSE / PSNR (§4)
def sse(ref: np.ndarray, test: np.ndarray, valid_height: int | None = None) -> list[int]:
    """Per-image sum of squared errors over the first valid_height rows
    (reading A13), exact Python ints.  Inputs (n, H, W)."""
    ref = np.asarray(ref, dtype=np.int64)
    test = np.asarray(test, dtype=np.int64)
    vh = ref.shape[1] if valid_height is None else valid_height
    d = ref[:, :vh, :] - test[:, :vh, :]
    return [int(v) for v in np.sum(d * d, axis=(1, 2))]


def psnr_from_sse(s: int, n_pixels: int, bit_depth: int) -> float:
    """PSNR = 10·log10(peak²·P/SSE), peak = 2^b - 1, +inf for SSE = 0
    (reading A7)."""
    if s == 0:
        return math.inf
    peak = (1 << bit_depth) - 1
    return 10.0 * math.log10(peak * peak * n_pixels / s)


# ----------------------------------------------------- image-level pipelines
def codec_images(imgs: np.ndarray, mode: str, r: int = 16, step: int = 16,
                 bit_depth: int = 8, valid_height: int | None = None) -> dict:
    """Whole-image §4 pipeline: blocks -> codec -> reassembled recon, per-image
    SSE and PSNR over the valid rows."""
    X = to_blocks(np.asarray(imgs, dtype=np.int64))
    if mode == "zonal":
        out = zonal_codec(X, r, bit_depth)
    elif mode == "uniform":
        out = uniform_codec(X, step, bit_depth)
    else:
        raise ValueError(mode)
    recon = from_blocks(out["recon"])
    vh = imgs.shape[1] if valid_height is None else valid_height
    s = sse(imgs, recon, vh)
    P = vh * imgs.shape[2]
    out.update({"recon_img": recon, "sse": s,
                "psnr": [psnr_from_sse(v, P, bit_depth) for v in s]})
    return out


def dct_zonal_images(imgs: np.ndarray, r: int, bit_depth: int = 8) -> dict:
    """Config-5 comparator: the exact DCT (brute-force cosines, reading A19)
    through the same zonal pipeline in float64: B = C·A·Cᵀ, keep r, A′ = Cᵀ·B′·C,
    round half away, clamp, PSNR."""
    C = tr.build_dct()
    X = to_blocks(np.asarray(imgs, dtype=np.int64)).astype(np.float64)
    Bc = (C @ X @ C.T) * tr.zonal_mask(r)
    A = C.T @ Bc @ C
    rec = clamp_pixels(round_half_away_float(A).astype(np.int64), bit_depth)
    recon = from_blocks(rec)
    s = sse(imgs, recon)
    P = imgs.shape[1] * imgs.shape[2]
    return {"recon_img": recon, "sse": s, "psnr": [psnr_from_sse(v, P, bit_depth) for v in s]}


def ape(psnr_approx: float, psnr_dct: float) -> float:
    """Absolute percentage error |PSNR_approx - PSNR_dct| / PSNR_dct x 100
    (PAPER.md:925-927)."""
    if math.isinf(psnr_approx) and math.isinf(psnr_dct):
        return 0.0
    return abs(psnr_approx - psnr_dct) / psnr_dct * 100.0
