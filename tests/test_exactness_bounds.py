"""Pins of the float32 exactness argument of the zonal kernels (DESIGN.md §5.2,
§5.3): the CUDA path evaluates the exact zonal numerator N = Tᵀ·(W ⊙ M_r ⊙ Z)·T
(W = 2304/(g_k·g_l)) in float32, which is exact only
while every value the transposed network forms is an integer (or, with the
+1152.5 rounding offset of the sweep, a half-integer) below 2^24 (2^23).

Every such value — each stage output of the transposed network of Eq. (1)
(M4ᵀ, M3ᵀ, M2ᵀ, M1ᵀ, taken from the oracle's factor list)
and every partial sum inside a stage row — is a LINEAR function L·X of the
image block, so its largest magnitude over all blocks X ∈ [0, maxpix]^256 is
exactly maxpix·max(Σ max(L, 0), −Σ min(L, 0)).  These tests compute that
maximum for the column pass and the row pass of the inverse and for the
running numerator N_r of the r-sweep, for every zonal r, and check the margins
the kernels rely on.  No GPU: this is a property of T, W and the zig-zag order."""
import itertools

import numpy as np
import pytest

from oracle import transform as tr

T = tr.build_T().astype(np.float64)
G = np.diag(T @ T.T)
W = 2304.0 / np.outer(G, G)
ORDER = [tuple(c) for c in tr.zigzag(16)]
# Z_kl as a linear functional of the 256 pixels: Z_kl = sum_ab T_ka T_lb X_ab
ZF = np.einsum("ka,lb->klab", T, T).reshape(16, 16, 256)


def _stage_values(F, xs, record):
    """y = F·x for a 0/±1 stage on vector-valued x; records every row output and
    every partial sum of 2+ of a row's terms (any accumulation order)."""
    ys = []
    for row in F:
        terms = [(int(row[j]), xs[j]) for j in range(len(row)) if row[j] != 0]
        for m in range(2, len(terms) + 1):
            for sub in itertools.combinations(terms, m):
                record.append(sum(s * v for s, v in sub))
        ys.append(sum(s * v for s, v in terms))
    return ys


def _inverse_network(ys, record):
    """x = Tᵀ·y through the transposed stages (oracle factor list, reversed)."""
    v = list(ys)
    for _, F in reversed(tr.factor_list()):
        v = _stage_values(F.T, v, record)
    return v


def _max_abs(vecs, maxpix):
    v = np.array(vecs)
    return maxpix * max(np.clip(v, 0, None).sum(1).max(), -np.clip(v, None, 0).sum(1).min())


def _zonal_inverse_extremes(r):
    """Largest |value| over 8-bit blocks in the column pass and the row pass of
    the zonal inverse with the first r zig-zag cells kept."""
    mask = np.zeros((16, 16))
    for k, l in ORDER[:r]:
        mask[k, l] = 1.0
    C = (W * mask)[:, :, None] * ZF
    rec1, rec2 = [], []
    U = np.zeros((16, 16, 256))
    for l in range(16):
        out = _inverse_network([C[k, l] for k in range(16)], rec1)
        for i in range(16):
            U[i, l] = out[i]
    rows = [_inverse_network([U[i, l] for l in range(16)], rec2) for i in range(16)]
    # the network reproduces N = Tᵀ·(W ⊙ M_r ⊙ Z)·T exactly (structure check)
    X = np.random.default_rng(r).integers(0, 256, 256).astype(np.float64)
    Z = T @ X.reshape(16, 16) @ T.T
    N = T.T @ (W * mask * Z) @ T
    assert np.allclose(np.array([[rows[i][j] @ X for j in range(16)] for i in range(16)]), N)
    return _max_abs(rec1, 255), _max_abs(rec2, 255)


def test_linear_bound_is_attained_on_the_paper_t():
    # the functional maximum is a real block: the all-255 block reaches Z_00 = 65280
    assert _max_abs([ZF[0, 0]], 255) == 65280.0
    assert _max_abs([ZF[1, 1]], 255) == 255.0 * np.clip(ZF[1, 1], 0, None).sum()


@pytest.mark.parametrize("r", [1, 6, 10, 16, 21, 28, 32, 36, 45, 64, 100, 128, 181, 200, 255, 256])
def test_zonal_inverse_values_fit_float32(r):
    p1, p2 = _zonal_inverse_extremes(r)
    # 8-bit (band kernel, tpb kernel, codec_warp zonal): integers + 1152 below 2^21
    assert p1 + 1152 < 2 ** 21 and p2 + 1152 < 2 ** 21
    # 10-bit (codec_warp zonal, 10-bit sweep): x 1023/255, half-integers below 2^23
    assert (p1 * 1023 / 255 + 1152.5) < 2 ** 23 and (p2 * 1023 / 255 + 1152.5) < 2 ** 23
    if r == 256:   # lossless: N = 2304·X
        assert p2 == 2304 * 255


def test_sweep_running_numerator_fits_float32():
    """N_r = N_{r-1} + W_kl·Z_kl·T_k⊗T_l for r = 1..256 (sweep.cu): every running
    value at every pixel, over every 8-bit block, stays below 2^21."""
    K = np.zeros((256, 256))   # N_r(i, j) = K[(i, j)] · X
    worst = 0.0
    for k, l in ORDER:
        v = np.outer(T[k], T[l]).ravel()
        K += W[k, l] * np.outer(v, v)
        worst = max(worst, 255 * max(np.clip(K, 0, None).sum(1).max(), -np.clip(K, None, 0).sum(1).min()))
    assert worst + 1152.5 < 2 ** 21
    assert worst * 1023 / 255 + 1152.5 < 2 ** 23
