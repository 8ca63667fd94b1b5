"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NONE of the method's arithmetic (no T, S, zig-zag, rounding or
PSNR): it only draws images.  It is the single place both sides take inputs from
("input recipe"), standing in for the paper's absent datasets
(45 USC-SIPI 512x512 images, Lena, the HEVC sequence — PAPER.md:856-860,
980-1017, 1357-1362) with the first-order Markov model the paper itself uses for
natural images (R[i,j] = rho^|i-j|, rho = 0.95).

Recipes (readings A11-A14 of DESIGN.md §3):
  * spatial field: w ~ N(0,1) of shape (H, W); filter along rows, then columns,
    with y_0 = w_0, y_j = rho·y_{j-1} + sqrt(1-rho²)·w_j (unit-variance
    stationary AR(1); covariance rho^(|di|+|dj|)).
  * 8-bit mapping: x = rint(128 + 40·(f - mean)/std), clip [0, 255], uint8.
  * 10-bit mapping: x = rint(512 + 160·(f - mean)/std), clip [0, 1023], int16.
  * config 1/2: image n of the batch uses default_rng(n) (cfg2 image 0 == cfg1).
  * config 3: E_t from default_rng(SeedSequence(1).spawn(n)[t]) (1080x1920,
    rho .95); F_0 = E_0, F_t = 0.9·F_{t-1} + sqrt(0.19)·E_t; per-frame 8-bit
    mapping; rows 1080..1087 := row 1079 (edge replication, reading A13).
  * config 4: frame f from default_rng(SeedSequence(2).spawn(1000)[f]),
    2160x3840, rho .95, 10-bit mapping.
  * config 5: seeds 100..163, rho .85 (100-115), .90 (116-131), .95 (132-147),
    .98 (148-163), 1024x1024, 8-bit mapping.
"""
from __future__ import annotations

import math
import os
from concurrent.futures import ProcessPoolExecutor

import numpy as np
from scipy.signal import lfilter

# ------------------------------------------------------------- the configs
CONFIGS = {
    1: dict(n=1, H=512, W=512, bit_depth=8, mode="zonal", r=16),
    2: dict(n=4096, H=512, W=512, bit_depth=8, mode="forward"),
    3: dict(n=600, H=1088, W=1920, valid_height=1080, bit_depth=8, mode="zonal", r=32),
    4: dict(n=1000, H=2160, W=3840, bit_depth=10, mode="uniform", step=16),
    5: dict(n=64, H=1024, W=1024, bit_depth=8, mode="sweep"),
}


def ar1_filter(w: np.ndarray, rho: float, axis: int) -> np.ndarray:
    """y_0 = w_0, y_j = rho·y_{j-1} + sqrt(1-rho²)·w_j along `axis`."""
    c = math.sqrt(1.0 - rho * rho)
    w = np.array(w, dtype=np.float64, copy=True)
    idx = [slice(None)] * w.ndim
    idx[axis] = 0
    w[tuple(idx)] /= c
    return lfilter([c], [1.0, -rho], w, axis=axis)


def ar1_field(rng: np.random.Generator, H: int, W: int, rho: float) -> np.ndarray:
    w = rng.standard_normal((H, W))
    return ar1_filter(ar1_filter(w, rho, axis=1), rho, axis=0)


def map_levels(f: np.ndarray, mean: float, std: float, lo: int, hi: int, dtype) -> np.ndarray:
    s = f.std()
    z = (f - f.mean()) / (s if s > 0 else 1.0)
    return np.clip(np.rint(mean + std * z), lo, hi).astype(dtype)


def map_u8(f: np.ndarray) -> np.ndarray:
    return map_levels(f, 128.0, 40.0, 0, 255, np.uint8)


def map_10bit(f: np.ndarray) -> np.ndarray:
    return map_levels(f, 512.0, 160.0, 0, 1023, np.int16)


# ------------------------------------------------------------ single items
def image_u8(seed: int, H: int = 512, W: int = 512, rho: float = 0.95) -> np.ndarray:
    """Configs 1, 2, 5: one AR(1) 8-bit image from default_rng(seed)."""
    return map_u8(ar1_field(np.random.default_rng(seed), H, W, rho))


def frame_10bit(f: int, H: int = 2160, W: int = 3840, seed: int = 2, total: int = 1000) -> np.ndarray:
    """Config 4: frame f (int16, values in [0, 1023])."""
    ss = np.random.SeedSequence(seed).spawn(total)[f]
    return map_10bit(ar1_field(np.random.default_rng(ss), H, W, 0.95))


def cfg5_rho(seed: int) -> float:
    return [0.85, 0.90, 0.95, 0.98][(seed - 100) // 16]


# ------------------------------------------------------------- batches
def _workers(n: int) -> int:
    try:
        cores = len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        cores = os.cpu_count() or 1
    return max(1, min(cores, n, 32))


def _img_job(args):
    seed, H, W, rho = args
    return image_u8(seed, H, W, rho)


def _f10_job(args):
    f, H, W, total = args
    return frame_10bit(f, H, W, total=total)


def batch_u8(seeds, H: int = 512, W: int = 512, rho=0.95, out: np.ndarray | None = None,
             workers: int | None = None) -> np.ndarray:
    """Stack of AR(1) 8-bit images, one per seed (parallel over host cores)."""
    seeds = list(seeds)
    rhos = [rho(s) if callable(rho) else rho for s in seeds]
    if out is None:
        out = np.empty((len(seeds), H, W), dtype=np.uint8)
    jobs = [(s, H, W, r) for s, r in zip(seeds, rhos)]
    nw = workers or _workers(len(jobs))
    if nw <= 1 or len(jobs) < 4:
        for i, j in enumerate(jobs):
            out[i] = _img_job(j)
    else:
        with ProcessPoolExecutor(nw) as ex:
            for i, im in enumerate(ex.map(_img_job, jobs, chunksize=max(1, len(jobs) // (4 * nw)))):
                out[i] = im
    return out


def frames_10bit(frame_ids, H: int = 2160, W: int = 3840, total: int = 1000,
                 out: np.ndarray | None = None, workers: int | None = None) -> np.ndarray:
    ids = list(frame_ids)
    if out is None:
        out = np.empty((len(ids), H, W), dtype=np.int16)
    jobs = [(f, H, W, total) for f in ids]
    nw = workers or _workers(len(jobs))
    if nw <= 1 or len(jobs) < 2:
        for i, j in enumerate(jobs):
            out[i] = _f10_job(j)
    else:
        with ProcessPoolExecutor(nw) as ex:
            for i, im in enumerate(ex.map(_f10_job, jobs)):
                out[i] = im
    return out


def _e_job(args):
    t, n, H, W, seed = args
    ss = np.random.SeedSequence(seed).spawn(n)[t]
    return ar1_field(np.random.default_rng(ss), H, W, 0.95).astype(np.float32)


def video_u8(n: int = 600, H: int = 1080, W: int = 1920, pad_to: int = 1088, seed: int = 1,
             workers: int | None = None) -> np.ndarray:
    """Config 3: spatial AR(1) fields with temporal AR(1) (rho_t = 0.9) drift,
    8-bit, rows [H, pad_to) replicated from row H-1."""
    out = np.empty((n, pad_to, W), dtype=np.uint8)
    nw = workers or _workers(n)
    prev = None
    a, b = 0.9, math.sqrt(1.0 - 0.81)
    jobs = [(t, n, H, W, seed) for t in range(n)]
    ex = ProcessPoolExecutor(nw) if nw > 1 and n > 1 else None
    try:
        it = ex.map(_e_job, jobs, chunksize=4) if ex else map(_e_job, jobs)
        for t, E in enumerate(it):
            F = E.astype(np.float64) if prev is None else a * prev + b * E.astype(np.float64)
            prev = F
            out[t, :H] = map_u8(F)
            out[t, H:] = out[t, H - 1]
    finally:
        if ex:
            ex.shutdown()
    return out


def config5_images(workers: int | None = None) -> np.ndarray:
    """Config 5: 64 images 1024x1024, seeds 100..163, rho by group of 16 (cfg5_rho)."""
    return batch_u8(range(100, 164), 1024, 1024, rho=cfg5_rho, workers=workers)


# ---------------------------------------------------- adversarial fixtures
def adversarial_u8(H: int = 64, W: int = 64, bit_depth: int = 8, seed: int = 7) -> np.ndarray:
    """Edge-case images: all-0, all-max, checkerboards, impulses, stripes,
    uniform noise over the full range (stack of 8 images)."""
    mx = (1 << bit_depth) - 1
    dt = np.uint8 if bit_depth == 8 else np.int16
    rng = np.random.default_rng(seed)
    yy, xx = np.mgrid[0:H, 0:W]
    imgs = [
        np.zeros((H, W)),
        np.full((H, W), mx),
        ((yy + xx) % 2) * mx,
        ((yy // 16 + xx // 16) % 2) * mx,
        np.where((yy % 16 == 3) & (xx % 16 == 11), mx, 0),
        (xx % 2) * mx,
        rng.integers(0, mx + 1, size=(H, W)),
        np.where(rng.random((H, W)) < 0.5, 0, mx),
    ]
    return np.stack([np.asarray(i).astype(dt) for i in imgs])
