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

// The exact levels of one block computed by its 16 lanes together (rare
// branch of the warp-per-block-pair codec): lane t runs the integer row
// network on row t of the block's ORIGINAL pixels (still in the stage), the
// rows meet in the scratch tile `qs` (int32, row pitch 20), lane l runs the
// column network on column l and decides its 16 levels exactly (uniform_fix),
// then overwrites the tile with them: qs[k·20 + l] = q_kl.  Returns whether
// lane l's column holds a nonzero level in an irrational cell (g_k != g_l).
// Every lane of the warp must call it (both blocks of the pair at once).
template <int ELEM>
__device__ __noinline__ bool block_levels_coop(const uint8_t* stage, int bb, int t, int step, int32_t* qs) {
    {
        int a0, a1;
        row_addr<ELEM>(bb, t, &a0, &a1);
        uint32_t w[4 * ELEM];
        load_px<ELEM>(stage, a0, a1, w);
        int32_t x[16], y[16];
        for (int j = 0; j < 16; ++j) x[j] = px_of<ELEM>(w, j);
        net_fwd(x, y);
        for (int l = 0; l < 16; ++l) qs[t * 20 + l] = y[l];
    }
    __syncwarp();
    const int l = t;
    {
        int32_t c[16], z[16];
        for (int k = 0; k < 16; ++k) c[k] = qs[k * 20 + l];
        net_fwd(c, z);
        __syncwarp();   // every lane has read its column before Z overwrites the tile
        for (int k = 0; k < 16; ++k) qs[k * 20 + l] = z[k];
    }
    bool irr = false;
    const float rstep = 1.0f / static_cast<float>(step);
    const int gl = g_of(l);
#pragma unroll 1
    for (int k = 0; k < 16; ++k) {   // rolled: this rare branch is kept small (instruction cache)
        const int32_t zk = qs[k * 20 + l];
        const uint32_t az = static_cast<uint32_t>(zk < 0 ? -zk : zk);
        const int gk = g_of(k);
        const int G = gk * gl;
        const uint64_t d2g = static_cast<uint64_t>(step) * step * G;
        // a float estimate (error < e·2^-21: rsqrtf within 2 ulp, two roundings); it
        // is the level unless its fraction lies within e·2^-20 of an integer, where
        // uniform_fix decides exactly (it corrects by one step)
        const float e = static_cast<float>(az) * rsqrtf(static_cast<float>(G)) * rstep + 0.5f;
        const float fl = floorf(e);
        const float fr = e - fl;
        const float mg = fmaf(e, 0x1p-20f, 0x1p-20f);
        int32_t m = static_cast<int32_t>(fl);
        if (fr < mg || fr > 1.0f - mg) m = uniform_fix(az, m, d2g);
        qs[k * 20 + l] = zk < 0 ? -m : m;
        irr |= m != 0 && gk != gl;
    }
    __syncwarp();
    return irr;
}

// The four integer components of 144·A′/Δ = J1 + J2·√2 + J3·√3 + J6·√6 (header
// of uexact.cuh) for row t of a block, computed by the block's 16 lanes from its
// exact levels qs[k·20 + l] (block_levels_coop): per component, lane l runs the
// transposed network down column l on the K-weighted levels, the columns meet
// in the scratch tile us (int32, pitch 20), lane t runs the transposed network
// along row t.  J[c][j]: c = 0, 1, 2, 3 for J1, J2 (√2), J3 (√3), J6 (√6).
// Every lane of the warp must call it.
__device__ __noinline__ void block_components_coop(const int32_t* qs, int32_t* us, int t, int32_t (&J)[4][16]) {
    const int e[3] = {3, 2, 3};    // 12·s_k = e·sqrt(rho2) per class (g = 16, 12, 8)
    const int r2[3] = {1, 3, 2};
    const int l = t;
    const int cl = uclass(l);
    // the K-weighted level of every cell of column l and the component it feeds
    int32_t wk[16], comp[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        const int ck = uclass(k);
        wk[k] = qs[k * 20 + l] * e[ck] * e[cl] * (ck == cl ? r2[ck] : 1);
        // J1 rational, J2 classes (16, 8): √2, J3 (16, 12): √3, J6 (12, 8): √6
        comp[k] = ck == cl ? 0 : (ck + cl == 2 ? 1 : (ck + cl == 1 ? 2 : 3));
    }
#pragma unroll 1
    for (int c = 0; c < 4; ++c) {   // rolled (rare branch, instruction cache); J is in local memory
        int32_t w[16], u[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) w[k] = comp[k] == c ? wk[k] : 0;
        net_inv(w, u);
#pragma unroll
        for (int i = 0; i < 16; ++i) us[i * 20 + l] = u[i];
        __syncwarp();
        int32_t r[16], jr[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) r[j] = us[t * 20 + j];
        net_inv(r, jr);
#pragma unroll
        for (int j = 0; j < 16; ++j) J[c][j] = jr[j];
        __syncwarp();
    }
}

// The exact branch of row t after the float64 row network (rare), given the
// row's float64 values `a`: pixels within 2^-20 of a .5 boundary decided
// exactly — by integer arithmetic on J1 when the block's levels are all in
// rational cells, else from the row's four components J (block_components_coop)
// — and clamped.
__device__ __noinline__ void exact_row_fix_levels(const double* a, const int32_t (*J)[16], bool rational,
                                                  int step, int maxpix, int* pix) {
    for (int j = 0; j < 16; ++j) {
        bool nr;
        int n0;
        round_f64(a[j], nr, n0);
        if (!nr) continue;
        int v;
        if (rational) {
            v = uniform_rational_floor(a[j], step);
        } else {
            const long long b0 = static_cast<long long>(step) * J[0][j] + 72 - 144LL * n0;
            v = sign_q23(b0, static_cast<long long>(step) * J[1][j], static_cast<long long>(step) * J[2][j],
                         static_cast<long long>(step) * J[3][j]) >= 0 ? n0 : n0 - 1;
        }
        pix[j] = min(max(v, 0), maxpix);
    }
}

}  // namespace
}  // namespace dct16a
