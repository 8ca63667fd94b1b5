"""Oracle, part 3: the paper's second image-quality measure, SSIM
("structural similarity index (SSIM) [Wang2004]").

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Plain numpy float64.

The paper gives no parameters; reading A21 takes the Wang et
al. 2004 defaults as SPEC.md:391-399 and 411 fix them: an 11x11 Gaussian
window with sigma = 1.5 normalised to unit sum, K1 = 0.01, K2 = 0.03, dynamic
range L = 2^b - 1, full resolution (no down-sampling), the mean of the SSIM map
over every window position lying fully inside the image ("valid" region) and
inside the first `valid_height` rows.
"""
from __future__ import annotations

import numpy as np

WIN = 11
SIGMA = 1.5
K1, K2 = 0.01, 0.03


def gaussian_window() -> np.ndarray:
    """w[u][v] ∝ exp(-((u-5)² + (v-5)²) / (2·1.5²)), sum 1 (Wang 2004)."""
    r = np.arange(WIN) - WIN // 2
    u, v = np.meshgrid(r, r, indexing="ij")
    w = np.exp(-(u * u + v * v) / (2.0 * SIGMA * SIGMA))
    return w / w.sum()


def _filter_valid(img: np.ndarray, w: np.ndarray) -> np.ndarray:
    """Σ_uv w[u][v]·img[i+u][j+v] for every fully contained window (float64)."""
    win = np.lib.stride_tricks.sliding_window_view(img, w.shape)
    return np.einsum("ijuv,uv->ij", win, w)


def ssim_map(ref: np.ndarray, test: np.ndarray, bit_depth: int = 8) -> np.ndarray:
    """The SSIM map of Wang et al. 2004, eq. (13), with local statistics from the
    Gaussian window: ((2μxμy + C1)(2σxy + C2)) / ((μx² + μy² + C1)(σx² + σy² + C2))."""
    x = np.asarray(ref, dtype=np.float64)
    y = np.asarray(test, dtype=np.float64)
    if x.shape != y.shape or min(x.shape) < WIN:
        raise ValueError("SSIM needs equal shapes of at least 11x11")
    L = float((1 << bit_depth) - 1)
    C1, C2 = (K1 * L) ** 2, (K2 * L) ** 2
    w = gaussian_window()
    mx, my = _filter_valid(x, w), _filter_valid(y, w)
    sxx = _filter_valid(x * x, w) - mx * mx
    syy = _filter_valid(y * y, w) - my * my
    sxy = _filter_valid(x * y, w) - mx * my
    return ((2 * mx * my + C1) * (2 * sxy + C2)) / ((mx * mx + my * my + C1) * (sxx + syy + C2))


def ssim(ref: np.ndarray, test: np.ndarray, bit_depth: int = 8, valid_height: int | None = None) -> list[float]:
    """Mean SSIM per image of (n, H, W) batches over the first valid_height rows."""
    ref = np.asarray(ref)
    test = np.asarray(test)
    vh = ref.shape[1] if valid_height is None else valid_height
    return [float(ssim_map(ref[i, :vh], test[i, :vh], bit_depth).mean()) for i in range(ref.shape[0])]


def ssim_bruteforce(ref: np.ndarray, test: np.ndarray, bit_depth: int = 8) -> float:
    """The same mean SSIM with Python loops over windows and taps (small-case pin)."""
    import math
    x = [[float(v) for v in row] for row in np.asarray(ref)]
    y = [[float(v) for v in row] for row in np.asarray(test)]
    H, W = len(x), len(x[0])
    g = [math.exp(-((u - 5) ** 2) / (2 * SIGMA * SIGMA)) for u in range(WIN)]
    s = sum(g[u] * g[v] for u in range(WIN) for v in range(WIN))
    L = float((1 << bit_depth) - 1)
    C1, C2 = (K1 * L) ** 2, (K2 * L) ** 2
    tot, cnt = 0.0, 0
    for i in range(H - WIN + 1):
        for j in range(W - WIN + 1):
            mx = my = exx = eyy = exy = 0.0
            for u in range(WIN):
                for v in range(WIN):
                    wt = g[u] * g[v] / s
                    a, b = x[i + u][j + v], y[i + u][j + v]
                    mx += wt * a
                    my += wt * b
                    exx += wt * a * a
                    eyy += wt * b * b
                    exy += wt * a * b
            vx, vy, cxy = exx - mx * mx, eyy - my * my, exy - mx * my
            tot += ((2 * mx * my + C1) * (2 * cxy + C2)) / ((mx * mx + my * my + C1) * (vx + vy + C2))
            cnt += 1
    return tot / cnt
