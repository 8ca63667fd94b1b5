// uexact_tile.cuh — the rare exact branches of the uniform fused codecs
// (codec_warp.cu, codec_uniform.cu) that re-read a block's ORIGINAL pixels
// from its TMA stage tile (tile128.cuh layout): exact levels by the integer
// network (reading A9) and the exact decision of a reconstruction pixel near a
// .5 boundary (reading A10, uexact.cuh).  Callers must not have overwritten
// the block's rows with the reconstruction yet.
#pragma once
#include <math.h>
#include <stdint.h>

#include "net16.cuh"
#include "quant.cuh"
#include "tables.cuh"
#include "tile128.cuh"
#include "uexact.cuh"

namespace dct16a {
namespace {

// Exact levels of one block recomputed from its pixels (rare branch): Z by the
// integer network, then the exact uniform decision (uniform_level/uniform_fix).
template <int ELEM>
__device__ __noinline__ void exact_levels_from_stage(const uint8_t* stage, int bb, int step, int32_t* q) {
    int32_t Y[16][16];
    for (int t = 0; t < 16; ++t) {
        int a0, a1;
        row_addr<ELEM>(bb, t, &a0, &a1);
        uint32_t w[4 * ELEM];
        load_px<ELEM>(stage, a0, a1, w);
        int32_t x[16], y[16];
        for (int j = 0; j < 16; ++j) x[j] = px_of<ELEM>(w, j);
        net_fwd(x, y);
        for (int l = 0; l < 16; ++l) Y[t][l] = y[l];
    }
    for (int l = 0; l < 16; ++l) {
        int32_t c[16], z[16];
        for (int t = 0; t < 16; ++t) c[t] = Y[t][l];
        net_fwd(c, z);
        for (int k = 0; k < 16; ++k) {
            const uint32_t az = static_cast<uint32_t>(z[k] < 0 ? -z[k] : z[k]);
            const uint64_t d2g = static_cast<uint64_t>(step) * step * (g_of(k) * g_of(l));
            const double e = static_cast<double>(az) / (step * sqrt(static_cast<double>(g_of(k) * g_of(l)))) + 0.5;
            const int32_t m = uniform_fix(az, static_cast<int32_t>(floor(e)), d2g);
            q[k * 16 + l] = z[k] < 0 ? -m : m;
        }
    }
}

// The exact branch of one lane's row t of block bb after the float64 row
// network (rare): `row` holds the row network's inputs; the row is recomputed,
// pixels near a .5 boundary decided exactly from the block's levels, every
// pixel clamped; returns the row's SSE and the packed reconstruction.
template <int ELEM>
__device__ __noinline__ uint32_t exact_row(const uint8_t* stage, int bb, const double* row, int t, int step,
                                           int maxpix, const uint32_t* orig, uint32_t* out) {
    double rr[16];
    for (int j = 0; j < 16; ++j) rr[j] = row[j];
    double a[16];
    net_inv(rr, a);
    int pix[16];
    bool any_near = false;
    for (int j = 0; j < 16; ++j) {
        bool nr;
        int n0;
        pix[j] = round_f64(a[j], nr, n0);
        any_near |= nr;
    }
    if (any_near) {
        int32_t qb[256];
        exact_levels_from_stage<ELEM>(stage, bb, step, qb);
        for (int j = 0; j < 16; ++j) {
            bool nr;
            int n0;
            round_f64(a[j], nr, n0);
            if (nr) pix[j] = uniform_exact_floor(qb, t, j, step, n0);
        }
    }
    uint32_t e = 0;
    for (int j = 0; j < 16; ++j) {
        const int p = min(max(pix[j], 0), maxpix);
        const int o = ELEM == 1 ? static_cast<int>((orig[j >> 2] >> (8 * (j & 3))) & 0xFFu)
                                : static_cast<int>((orig[j >> 1] >> (16 * (j & 1))) & 0xFFFFu);
        e += static_cast<uint32_t>((p - o) * (p - o));
        pix[j] = p;
    }
    for (int q = 0; q < 4 * ELEM; ++q) {
        out[q] = ELEM == 1 ? (pix[4 * q] | (pix[4 * q + 1] << 8) | (pix[4 * q + 2] << 16) | (pix[4 * q + 3] << 24))
                           : (pix[2 * q] | (pix[2 * q + 1] << 16));
    }
    return e;
}

// Rare branch of the uniform rounding: row t of the block has a pixel within
// 2^-20 of a .5 boundary.  Recompute the row from the transposition tile (still
// intact), flag the near pixels again and decide them exactly from the levels.
template <int ELEM>
__device__ __noinline__ void exact_row_fix(const uint8_t* stage, int bb, const double* urow, int t, int step,
                                           int maxpix, int* pix) {
    double rr[16], a[16];
    for (int j = 0; j < 16; ++j) rr[j] = urow[j];
    net_inv(rr, a);
    int32_t qb[256];
    exact_levels_from_stage<ELEM>(stage, bb, step, qb);
    for (int j = 0; j < 16; ++j) {
        bool nr;
        int n0;
        round_f64(a[j], nr, n0);
        if (nr) pix[j] = min(max(uniform_exact_floor(qb, t, j, step, n0), 0), maxpix);
    }
}

}  // namespace
}  // namespace dct16a
