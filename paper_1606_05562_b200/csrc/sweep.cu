// sweep.cu — the zonal codec for a whole range of retained-coefficient counts
// r in one pass over the images (config 5: the r-sweep of the paper's image
// compression experiment, Figs. 1-2; reading A4 zig-zag).
//
// With S folded into the weights the exact reconstruction
// numerator of dct16a_codec is N_r = Tᵀ·(W ⊙ M_r ⊙ Z)·T, and M_r differs from
// M_{r-1} in the single zig-zag cell (k, l) of rank r-1, so
//     N_r = N_{r-1} + W_kl·Z_kl · T_k ⊗ T_l        (outer product of rows of T).
// Every step is a rank-1 update of the 16x16 numerator followed by the same
// rounding (reading A6) and SSE as the fused codec; the pixels for every r are
// therefore byte-identical to dct16a_codec with that r.
//
// Layout: one warp holds a block pair, lane = row i of its block (as in
// codec_warp.cu): TMA tile ring in the 128-byte swizzle (tile128.cuh), row
// pass, smem transposition, column pass (lane = column l) producing W ⊙ Z into
// smem, then the sweep with lane = row i: N[i][:] += (W·Z_kl·T_ki)·T_l[:] in
// float32 (exact: half-integers below 2^21 for 8-bit and 2^23 for 10-bit
// input, the worst case over all blocks and all r pinned by tests/
// test_exactness_bounds.py; the +1152.5 rounding offset rides
// in N from the start; two columns per FFMA2; N is held as N·2^-35),
// pixel = floor(N/2304) by one round-down multiply into the subnormal range
// whose bits are the integer (8-bit; zonal_band.cu) or one round-down FMA onto
// 2^23 (10-bit), clamp,
// squared error in float32 (exact below 2^24 per row), one REDUX per r and a
// shared-memory 64-bit atomic into the warp's per-r SSE, flushed to global per
// image.
#include <cuda.h>
#include <stdint.h>

#include "internal.h"
#include "net16.cuh"
#include "ptx.cuh"
#include "quant.cuh"
#include "tables.cuh"
#include "tile128.cuh"

namespace dct16a {
namespace {

#ifndef DCT16A_SWEEP_UNROLL
#define DCT16A_SWEEP_UNROLL 8
#endif
constexpr int kSweepUnroll = DCT16A_SWEEP_UNROLL;   // measured r-loop unroll
constexpr int kSWarps = 4;    // warps per CTA

// zig-zag order as a table: kZZ[r] = 16·k + l of the cell with rank r (reading A4)
struct ZZTable {
    uint8_t v[256];
};
constexpr ZZTable make_zz() {
    ZZTable t{};
    for (int k = 0; k < 16; ++k)
        for (int l = 0; l < 16; ++l) t.v[zigzag_rank(k, l)] = static_cast<uint8_t>(16 * k + l);
    return t;
}
__constant__ ZZTable c_zz = make_zz();

template <int ELEM>
struct SCfg {
    // TMA ring depth per warp: every tile is 256 rank-1 steps of work, so two stages
    // hide the loads for 8-bit input (shared memory for 3 CTAs with four rows per lane);
    // 10-bit keeps three (0.87 against 0.93 ms)
    static constexpr int kSStages = ELEM == 1 ? 2 : 3;
    static constexpr int kStageBytes = 16 * kWTile * 16 * ELEM;
    // rows per lane in the sweep: every lane carries row t of several blocks (four for
    // 8-bit input: the whole 8-block tile; two for 10-bit), so each step's operands
    // (zig-zag cell, T_ki, the row T_l) are fetched once for all of them (config 5:
    // 2.32 ms with one row, 2.00 with two, 1.86 with four; 10-bit 0.96 -> 0.87 ms with two)
    static constexpr int kRPL = ELEM == 1 ? 4 : 2;
    // per warp: stages | Y transposition (2 x 336 floats) + W⊙Z (2·kRPL x 257 floats) | SSE[256] u64
    static constexpr int kYBytes = 3072, kZBytes = 2048 * kRPL, kSseBytes = 2048;
    static constexpr int kWarpBytes = kSStages * kStageBytes + kYBytes + kZBytes + kSseBytes;
    static_assert(kWarpBytes % 1024 == 0, "stages must stay 1024-byte aligned");
    static constexpr int kTBytes = 1024;   // T as floats, shared by the CTA
    static constexpr int kSmem = 1024 + kSWarps * kWarpBytes + kTBytes + kSWarps * kSStages * 8;
    static constexpr int kFit = (227 * 1024) / (kSmem + 1024);
    static constexpr int kCtasPerSm = kFit < 4 ? kFit : 4;
};

struct SParams {
    int W, BX, BY, VH, tiles_per_strip, maxpix;
    long long n_tiles, chunk;
    int r_first, r_count, r_last;
};

}  // namespace

template <int ELEM>
__global__ void __launch_bounds__(kSWarps * 32, SCfg<ELEM>::kCtasPerSm)
    sweep_kernel(const __grid_constant__ CUtensorMap tin, unsigned long long* __restrict__ sse, const SParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = walign1024(smem_raw);
    using Cfg = SCfg<ELEM>;
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int h = lane >> 4, t = lane & 15;
    uint8_t* wbase = smem + warp * Cfg::kWarpBytes;
    float* ty = reinterpret_cast<float*>(wbase + Cfg::kSStages * Cfg::kStageBytes) + h * (16 * 20 + 16);
    // W⊙Z of the block pair right after the Y tile (2 x 336 floats); the second block
    // starts 257 floats later so the two half-warps' broadcasts hit different banks
    float* wz = reinterpret_cast<float*>(wbase + Cfg::kSStages * Cfg::kStageBytes) + 2 * 336 + h * 257;
    unsigned long long* ssew =
        reinterpret_cast<unsigned long long*>(wbase + Cfg::kSStages * Cfg::kStageBytes + Cfg::kYBytes + Cfg::kZBytes);
    float* Ts = reinterpret_cast<float*>(smem + kSWarps * Cfg::kWarpBytes);   // Ts[k*16 + i] = T[k][i]
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kSWarps * Cfg::kWarpBytes + Cfg::kTBytes) + warp * Cfg::kSStages;

    // T from the network of Eq. (1): column i = net_fwd(e_i)
    if (threadIdx.x < 16) {
        float x[16], y[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) x[j] = j == static_cast<int>(threadIdx.x) ? 1.0f : 0.0f;
        net_fwd(x, y);
#pragma unroll
        for (int k = 0; k < 16; ++k) Ts[k * 16 + threadIdx.x] = y[k];
    }
    for (int i = lane; i < 256; i += 32) ssew[i] = 0;

    const long long gw = static_cast<long long>(blockIdx.x) * kSWarps + warp;
    const long long t0 = gw * p.chunk;
    long long t1 = t0 + p.chunk;
    if (t1 > p.n_tiles) t1 = p.n_tiles;
    const uint64_t pol = policy_evict_first();
    if (lane == 0) {
        for (int s = 0; s < Cfg::kSStages; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
        prefetch_tmap(&tin);
        TileCursor ic;
        ic.init(p, t0);
        for (int s = 0; s < Cfg::kSStages - 1; ++s) {
            if (t0 + s < t1) w_issue_at<ELEM>(&tin, p, ic, wbase + s * Cfg::kStageBytes, &bars[s], pol);
            ic.advance(p);
        }
    }
    __syncthreads();

    // per-lane weights of column l = t by class of k: W = 2304/(g_k·g_l)
    const int l = t;
    // N is carried as N·2^-35 (exact: half-integers below 2^23 times a power of two),
    // so the 8-bit rounding can land its integer in the subnormal bits (header)
    const float w16 = static_cast<float>(2304 / (16 * g_of(l))) * 0x1p-35f;
    const float w12 = static_cast<float>(2304 / (12 * g_of(l))) * 0x1p-35f;
    const float w8 = static_cast<float>(2304 / (8 * g_of(l))) * 0x1p-35f;
    const float inv2304 = 0x1p35f / 2304.0f;   // 10-bit: floor onto 2^23 of N·2^-35 · 2^35/2304
    const float top = 8388608.0f + static_cast<float>(p.maxpix);

    int cur_n = -1;
    int it = 0;
    TileCursor cc, nc;   // the tile being consumed and the one kSStages - 1 ahead (next to issue)
    cc.init(p, t0);
    nc.init(p, t0 + Cfg::kSStages - 1);
    for (long long tix = t0; tix < t1; ++tix, ++it, cc.advance(p), nc.advance(p)) {
        const int s = it % Cfg::kSStages;
        uint8_t* stage = wbase + s * Cfg::kStageBytes;
        mbar_wait(&bars[s], (it / Cfg::kSStages) & 1);
        const int n = cc.n, by = cc.by, x0 = cc.x0();
        if (n != cur_n) {   // flush the per-r SSE of the previous image (warp-uniform)
            __syncwarp();
            if (cur_n >= 0)
                for (int i = lane; i < p.r_count; i += 32) {
                    if (ssew[i]) atomicAdd(sse + static_cast<long long>(cur_n) * p.r_count + i, ssew[i]);
                    ssew[i] = 0;
                }
            __syncwarp();
            cur_n = n;
        }
        const int nb = min(kWTile, p.BX - x0 / 16);
        const bool row_valid = by * 16 + t < p.VH;
        constexpr int RPL = Cfg::kRPL;
#pragma unroll 1
        for (int grp = 0; 2 * RPL * grp < nb; ++grp) {
            // lane (h, t): row t of blocks 2·RPL·grp + 2u + h, u < RPL
            bool contributes[RPL];
            float xs[RPL][ELEM == 2 ? 16 : 1];   // 10-bit: 2^23 + x[i][j], the SSE reference in the magic-float domain
            uint32_t xw[RPL][4];                 // 8-bit: the packed original row (vabsdiff4/dp4a reference)
#pragma unroll
            for (int u = 0; u < RPL; ++u) {
                const int bb = 2 * RPL * grp + 2 * u + h;
                contributes[u] = bb < nb && row_valid;
                int a0, a1;
                row_addr<ELEM>(bb, t, &a0, &a1);
                {
                    uint32_t w[4 * ELEM];
                    load_px<ELEM>(stage, a0, a1, w);
                    if (ELEM == 1) {
#pragma unroll
                        for (int q = 0; q < 4; ++q) xw[u][q] = w[q];
                    }
                    float x[16], y[16];
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        x[j] = px_float<ELEM>(w, j);
                        if constexpr (ELEM == 2) xs[u][j] = 8388608.0f + x[j];
                    }
                    net_fwd(x, y);
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        *reinterpret_cast<float4*>(ty + t * 20 + 4 * q) = make_float4(y[4 * q], y[4 * q + 1], y[4 * q + 2], y[4 * q + 3]);
                }
                __syncwarp();
                {
                    float col[16], z[16];
#pragma unroll
                    for (int k = 0; k < 16; ++k) col[k] = ty[k * 20 + l];
                    net_fwd(col, z);
                    float* wzu = wz + u * 2 * 257;
#pragma unroll
                    for (int k = 0; k < 16; ++k)
                        wzu[k * 16 + l] = z[k] * (g_of(k) == 16 ? w16 : (g_of(k) == 12 ? w12 : w8));
                }
                __syncwarp();
            }
            // ---- the sweep, lane = row i = t of each of its RPL blocks
            // N[u][i][2m], N[u][i][2m+1] as one float2: the update and the rounding are FFMA2
            float2 N[RPL][8];
#pragma unroll
            for (int u = 0; u < RPL; ++u)
#pragma unroll
                for (int m = 0; m < 8; ++m) N[u][m] = make_float2(1152.5f * 0x1p-35f, 1152.5f * 0x1p-35f);
            // operands of the rank-1 step r (zig-zag cell of rank r-1), prefetched one step ahead:
            // W⊙Z_kl·T_ki of each block (T_ki shared: row i = t of every block) and the row T_l
            float sv[RPL];
            float4 tq[4];
            auto fetch = [&](int r, float (&s_out)[RPL], float4 (&t_out)[4]) {
                const int kl = c_zz.v[min(r, 256) - 1];
                const float tk = Ts[(kl >> 4) * 16 + t];
#pragma unroll
                for (int u = 0; u < RPL; ++u) s_out[u] = wz[u * 2 * 257 + kl] * tk;
                const float4* tr = reinterpret_cast<const float4*>(Ts + (kl & 15) * 16);
#pragma unroll
                for (int q = 0; q < 4; ++q) t_out[q] = tr[q];
            };
            auto update = [&]() {
#pragma unroll
                for (int u = 0; u < RPL; ++u) {
                    const float2 s2 = make_float2(sv[u], sv[u]);
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        N[u][2 * q] = __ffma2_rn(s2, make_float2(tq[q].x, tq[q].y), N[u][2 * q]);
                        N[u][2 * q + 1] = __ffma2_rn(s2, make_float2(tq[q].z, tq[q].w), N[u][2 * q + 1]);
                    }
                }
            };
            auto rotate = [&](const float (&svn)[RPL], const float4 (&tqn)[4]) {
#pragma unroll
                for (int u = 0; u < RPL; ++u) sv[u] = svn[u];
#pragma unroll
                for (int q = 0; q < 4; ++q) tq[q] = tqn[q];
            };
            const float2 inv2 = make_float2(inv2304, inv2304), m2 = make_float2(8388608.0f, 8388608.0f);
            const float2 pix2 = make_float2(0x1p-114f / 2304.0f, 0x1p-114f / 2304.0f);
            fetch(1, sv, tq);
#pragma unroll 1
            for (int r = 1; r < p.r_first; ++r) {   // below the requested range: update only
                float svn[RPL];
                float4 tqn[4];
                fetch(r + 1, svn, tqn);
                update();
                rotate(svn, tqn);
            }
#pragma unroll kSweepUnroll
            for (int r = p.r_first; r <= p.r_last; ++r) {
                float svn[RPL];
                float4 tqn[4];
                fetch(r + 1, svn, tqn);
                update();
                unsigned ei = 0;
#pragma unroll
                for (int u = 0; u < RPL; ++u) {
                    unsigned eu;
                    if (ELEM == 1) {
                        // (N·2^-35)·fl(2^-114/2304) rounded down to the subnormal grid: the bits
                        // are floor(N·fl(1/2304)) (negative -> sign bit -> 0); cvt.pack.sat clamps
                        // to [0, 255] and packs 4 pixels, vabsdiff4 + dp4a square and sum
                        eu = 0;
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const float2 f0 = fmul2_rd_keep_subnormal(N[u][2 * q], pix2),
                                         f1 = fmul2_rd_keep_subnormal(N[u][2 * q + 1], pix2);
                            const int v[4] = {__float_as_int(f0.x), __float_as_int(f0.y), __float_as_int(f1.x),
                                              __float_as_int(f1.y)};
                            const uint32_t pk = pack2_sat_u8(v[1], v[0], pack2_sat_u8(v[3], v[2], 0u));
                            const uint32_t d = __vabsdiffu4(pk, xw[u][q]);
                            eu = __dp4a(d, d, eu);
                        }
                    } else {
                        // floor((N + 1152.5)/2304) by one round-down FMA onto 2^23 (exact, header),
                        // float32 clamp and squared error (exact below 2^24 per row)
                        float2 e2 = make_float2(0.0f, 0.0f);
#pragma unroll
                        for (int m = 0; m < 8; ++m) {
                            const float2 f = __ffma2_rd(N[u][m], inv2, m2);
                            const float2 fc = make_float2(fminf(fmaxf(f.x, 8388608.0f), top), fminf(fmaxf(f.y, 8388608.0f), top));
                            const float2 d = __fadd2_rn(fc, make_float2(-xs[u][2 * m], -xs[u][2 * m + 1]));
                            e2 = __ffma2_rn(d, d, e2);
                        }
                        eu = __float2uint_rn(e2.x + e2.y);
                    }
                    ei += contributes[u] ? eu : 0u;
                }
                const unsigned tot = __reduce_add_sync(0xffffffffu, ei);
                if (lane == 0) ssew[r - p.r_first] += tot;   // this warp's own accumulator: no atomic
                rotate(svn, tqn);
            }
            __syncwarp();
        }
        if (lane == 0) {
            const long long nt = tix + Cfg::kSStages - 1;
            if (nt < t1) w_issue_at<ELEM>(&tin, p, nc, wbase + ((it + Cfg::kSStages - 1) % Cfg::kSStages) * Cfg::kStageBytes,
                                       &bars[(it + Cfg::kSStages - 1) % Cfg::kSStages], pol);
        }
        __syncwarp();
    }
    __syncwarp();
    if (cur_n >= 0)
        for (int i = lane; i < p.r_count; i += 32)
            if (ssew[i]) atomicAdd(sse + static_cast<long long>(cur_n) * p.r_count + i, ssew[i]);
}

namespace {

template <int ELEM>
int launch_sweep_t(const void* src, const Geom& g, int r_first, int r_count, uint64_t* sse, cudaStream_t st) {
    using Cfg = SCfg<ELEM>;
    CUtensorMap tin;
    const uint64_t dims[3] = {uint64_t(g.W), uint64_t(g.H), uint64_t(g.N)};
    const uint64_t strides[2] = {uint64_t(g.pitch), uint64_t(g.istride)};
    const uint32_t box[3] = {uint32_t(128 / ELEM), 16u, 1u};
    if (encode_tiled(&tin, ELEM == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, src, dims,
                     strides, box, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B))
        return DCT16A_ECUDA;
    SParams p{};
    p.W = g.W;
    p.BX = g.BX;
    p.BY = g.BY;
    p.VH = g.VH;
    p.tiles_per_strip = (g.BX + kWTile - 1) / kWTile;
    p.maxpix = (1 << g.bits) - 1;
    p.n_tiles = static_cast<long long>(g.N) * g.BY * p.tiles_per_strip;
    p.r_first = r_first;
    p.r_count = r_count;
    p.r_last = r_first + r_count - 1;
    if (int e = smem_optin(reinterpret_cast<const void*>(sweep_kernel<ELEM>), Cfg::kSmem)) return e;
    long long warps = static_cast<long long>(num_sms()) * Cfg::kCtasPerSm * kSWarps;
    if (warps > p.n_tiles) warps = p.n_tiles;
    p.chunk = (p.n_tiles + warps - 1) / warps;
    const long long grid = (warps + kSWarps - 1) / kSWarps;
    sweep_kernel<ELEM><<<static_cast<unsigned>(grid), kSWarps * 32, Cfg::kSmem, st>>>(
        tin, reinterpret_cast<unsigned long long*>(sse), p);
    return static_cast<int>(cudaGetLastError());
}

}  // namespace

int launch_sweep(const void* src, const Geom& g, int r_first, int r_count, uint64_t* sse, double* psnr,
                 cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(sse, 0, sizeof(uint64_t) * g.N * r_count, st);
    if (e) return static_cast<int>(e);
    const int rc = g.elem == 1 ? launch_sweep_t<1>(src, g, r_first, r_count, sse, st)
                               : launch_sweep_t<2>(src, g, r_first, r_count, sse, st);
    if (rc) return rc;
    return launch_psnr_finish(g, static_cast<long long>(g.N) * r_count, sse, psnr, st);
}

}  // namespace dct16a
