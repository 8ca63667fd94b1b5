// codec_uniform.cu — the fused codec with the uniform quantiser (config 4):
// forward, quantisation with S folded in (PAPER.md:305-344,
// reading A9), inverse in float64 (reading A10), round half
// away / clamp (reading A6), per-image SSE, for 8- and
// 10-bit pixels.
//
// EXPERIMENT BUILD ONLY (-DDCT16A_EXPERIMENTS, codec path 4): measured slower
// than codec_warp.cu on config 4 (profiles/r02_config4_packed_lanes.md): the
// packing halves the float32 forward but adds register moves, a per-lane Z
// buffer and per-tile overheads, at a lower issue rate.
//
// Work unit: a warp takes a tile of 8 blocks (16 rows x 128 px, tile128.cuh)
// from its TMA ring and runs it as two quads of 4 blocks.  Lane (h, t) owns
// row t (then column t) of the block PAIR (A, B) = (4q + 2h, 4q + 2h + 1):
// the two blocks travel together as the two halves of a float2, so every
// float32 step is one packed FADD2/FFMA2 for both blocks.
// * Forward, float32 (exact: every partial sum is an integer < 2^19, V9):
//   pixels -> float by I2F.U8/U16 with byte/half selectors, row network of
//   Eq. (1) on F2 values, per-half-warp transposition tile (the paper's
//   transposition buffer; 128-byte rows, 16-byte chunks
//   XOR-swizzled by the row), column network.
// * Quantiser (reading A9), both blocks at once: e = |Z|·c + 1/2 + δ by one
//   FFMA2 (|.| is an operand modifier) and one round-down FADD2 onto the magic
//   1.5·2^(23-F): the float's bits are magic + m·2^F + F fraction bits.  δ
//   (> the float error, below the spacing of the rational cells) makes the
//   rational cells — the only ones with exact ties — exact; an irrational cell
//   whose fraction falls in [0, wbits·2^-F) is re-decided in integers
//   (uniform_fix, rare).
// * Level -> float64: the high word of d = 2^20 + m is (bits >> F) + const:
//   ONE IMAD.HI; c = d·w − 2^20·w (one DFMA, w = Δ·s_k·s_l, the product
//   2^20·w exact) is the S-scaled level, correctly rounded; the sign of Z
//   flips c's sign bit.
// * Inverse, float64, one block of the pair after the other: column network,
//   transposition through the same smem tile (doubles, swizzled), row network.
// * Rounding: one round-down DADD onto 1.5·2^20 + 1/2 + 2^-20 puts
//   0x41380000 + floor(A′ + 1/2) in the high word and the fraction (+2^-20) in
//   the low word; low word < 2^-19·2^32 flags a value within 2^-20 of a .5
//   boundary, a high word outside [0x41380000, 0x41380000 + maxpix] a pixel to
//   clamp: either sends the lane to the exact branch (rare).  Otherwise the
//   pixel is the high word's low half (packed by PRMT) and the squared error
//   is (hi - (0x41380000 + x))² by one IMAD.
// * SSE per row in 32 bits, one 64-bit atomic per warp and image; the
//   reconstruction overwrites the stage tile in place and leaves by TMA store.
// * Schedule: persistent warps claim runs of tiles (sched.cuh).
#ifdef DCT16A_EXPERIMENTS
#include <cuda.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>

#include "internal.h"
#include "net16.cuh"
#include "pack2.cuh"
#include "ptx.cuh"
#include "quant.cuh"
#include "sched.cuh"
#include "tables.cuh"
#include "tile128.cuh"
#include "uexact.cuh"
#include "uexact_tile.cuh"

namespace dct16a {
namespace {

#ifndef DCT16A_CU_STAGES
#define DCT16A_CU_STAGES 2
#endif
#ifndef DCT16A_CU_CTAS
#define DCT16A_CU_CTAS 3
#endif
#ifndef DCT16A_CU_CLAIM
#define DCT16A_CU_CLAIM 4
#endif
constexpr int kUWarps = 4;                  // warps per CTA
constexpr int kUStages = DCT16A_CU_STAGES;  // TMA ring depth per warp
constexpr int kUHalf = 2048;                // transposition tile per half-warp: 16 x 16 x 8 B
constexpr int kUXpose = 2 * kUHalf;
constexpr int kUZbuf = 32 * 128;            // per lane: Z of its column for both blocks (2 x 16 floats)
constexpr int kUClaim = DCT16A_CU_CLAIM;

template <int ELEM>
struct UCfg {
    static constexpr int kStageBytes = 16 * kWTile * 16 * ELEM;   // 2 KB (u8) / 4 KB (u16)
    static constexpr int kWarpBytes = kUStages * kStageBytes + kUXpose + kUZbuf;
    static_assert(kWarpBytes % 1024 == 0, "stages must stay 1024-byte aligned");
    // + per warp: kUStages mbarriers, the coordinates (n, by, tb, valid) of each
    // stage's tile and lane 0's claim state; per CTA: the (w, k) float64 pairs of
    // the level conversion for every column and class (kept out of registers)
    static constexpr int kSmem = 1024 + kUWarps * kWarpBytes + kUWarps * kUStages * (8 + 16) + kUWarps * 32 + 16 * 3 * 16;
    static constexpr int kFit = (227 * 1024) / (kSmem + 1024);
    static constexpr int kCtasPerSm = kFit < DCT16A_CU_CTAS ? kFit : DCT16A_CU_CTAS;
};

constexpr int kMaxPeers = 8;
__device__ unsigned long long g_cu_sched[kSchedSlots][2];

struct UParams {
    int W, BX, BY, VH, tiles_per_strip, maxpix;
    long long n_tiles;
    int slot, total_warps, claim;   // tile scheduler (sched.cuh; slot -1 = static), tiles per claim
    int has_recon;
    int n_peers, multicast;         // fused SSE all-reduce (as codec_warp.cu)
    long long frame_offset;
    unsigned long long* peers[kMaxPeers];
    int step, F;
    float cq[16][3];                // 1/(Δ·sqrt(g_k·g_l)) for column l and class of k (float, host-rounded)
    uint32_t wbits;                 // window: fraction (low F bits) < wbits -> exact decision
    uint32_t fmask;                 // (1 << F) - 1
    uint32_t hi_mul, hi_add;        // high word of 2^20 + m = umulhi(bits, hi_mul) + hi_add
    float magic_f, half_delta;
    double w[48];                   // Δ·s_k·s_l, index 3·l + class of k
};

// lane 0's claim state (shared memory: the other lanes need no registers for it)
struct WarpClaims {
    long long next, end, k;   // tiles [next, end) of the claim in progress; claims made (static schedule)
    int n, by, tb, pad;       // tile cursor of `next`
};

// rounding: 0x41380000 is the high word of 1.5·2^20
constexpr uint32_t kRoundHi = 0x41380000u;
// 1.5·2^20 + 1/2 + 2^-20: the low word then carries frac + 2^-20 (see header)
__device__ __forceinline__ double round_magic() { return 1572864.5 + 0x1p-20; }

// Add one image's SSE (as codec_warp.cu: local, multicast, or peer atomics).
__device__ __forceinline__ void flush_sse_u(unsigned long long* sse, const UParams& p, int n, unsigned long long v) {
    if (p.n_peers == 0) {
        atomicAdd(sse + n, v);
        return;
    }
    if (p.multicast) {
        asm volatile("multimem.red.relaxed.sys.global.add.u64 [%0], %1;" ::"l"(p.peers[0] + p.frame_offset + n), "l"(v)
                     : "memory");
        return;
    }
    for (int q = 0; q < p.n_peers; ++q) atomicAdd_system(p.peers[q] + p.frame_offset + n, v);
}

// swizzled transposition tiles (per half-warp, 16 rows of 128 bytes): element
// (r, c) of 8-byte entries lives in chunk (c >> 1) ^ (r & 7) of row r
__device__ __forceinline__ int xp_off(int r, int c) { return r * 128 + ((((c >> 1) ^ (r & 7))) << 4) + ((c & 1) << 3); }

// Pixel j of a row as float (I2F with a byte / half selector).
template <int ELEM>
__device__ __forceinline__ float px_f(const uint32_t (&w)[4 * ELEM], int j) {
    if (ELEM == 1) return static_cast<float>((w[j >> 2] >> (8 * (j & 3))) & 0xFFu);
    return static_cast<float>((w[j >> 1] >> (16 * (j & 1))) & 0xFFFFu);
}

// Exact level of a flagged coefficient (rare): returns the S-scaled float64 input.
__device__ __forceinline__ double exact_level_input(float z, uint32_t bits, float magic, int F, int step, int G, double w) {
    const uint32_t az = static_cast<uint32_t>(fabsf(z));
    const int32_t m0 = static_cast<int32_t>((bits - __float_as_uint(magic)) >> F);
    const int32_t m = uniform_fix(az, m0, static_cast<uint64_t>(step) * step * G);
    const double c = static_cast<double>(m) * w;
    return z < 0.0f ? -c : c;
}

}  // namespace

template <int ELEM>
__global__ void __launch_bounds__(kUWarps * 32, UCfg<ELEM>::kCtasPerSm)
    codec_uniform_kernel(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout,
                         unsigned long long* __restrict__ sse, const UParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = walign1024(smem_raw);
    using Cfg = UCfg<ELEM>;
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int h = lane >> 4, t = lane & 15;
    uint8_t* wbase = smem + warp * Cfg::kWarpBytes;
    uint8_t* xph = wbase + kUStages * Cfg::kStageBytes + h * kUHalf;   // this half-warp's transposition tile
    uint8_t* zb = wbase + kUStages * Cfg::kStageBytes + kUXpose + lane * 128;   // this lane's Z buffer
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kUWarps * Cfg::kWarpBytes) + warp * kUStages;
    int4* coords = reinterpret_cast<int4*>(smem + kUWarps * Cfg::kWarpBytes + kUWarps * kUStages * 8) +
                   warp * kUStages;
    WarpClaims* wcl = reinterpret_cast<WarpClaims*>(coords + (kUWarps - warp) * kUStages) + warp;
    double2* wktab = reinterpret_cast<double2*>(reinterpret_cast<uint8_t*>(coords + (kUWarps - warp) * kUStages) +
                                                kUWarps * sizeof(WarpClaims));
    const uint64_t pol = policy_evict_first();
    unsigned long long* sched = p.slot >= 0 ? g_cu_sched[p.slot] : nullptr;

    // claim the next tile and issue its load into stage st (lane 0; state in smem)
    auto issue_next = [&](int st) {
        WarpClaims c = *wcl;
        if (c.next == c.end) {
            const long long idx = sched ? static_cast<long long>(atomicAdd(sched, 1ull))
                                        : static_cast<long long>(blockIdx.x) * kUWarps + warp +
                                              (c.k++) * static_cast<long long>(gridDim.x) * kUWarps;
            const long long first = idx * p.claim;
            c.next = first;
            c.end = first < p.n_tiles ? min(first + p.claim, p.n_tiles) : first;
            if (first < p.n_tiles) {
                TileCursor ic;
                ic.init(p, first);
                c.n = ic.n;
                c.by = ic.by;
                c.tb = ic.tb;
            }
        }
        if (c.next < c.end) {
            TileCursor ic;
            ic.n = c.n;
            ic.by = c.by;
            ic.tb = c.tb;
            coords[st] = make_int4(ic.n, ic.by, ic.tb, 1);
            w_issue_at<ELEM>(&tin, p, ic, wbase + st * Cfg::kStageBytes, &bars[st], pol);
            ++c.next;
            ic.advance(p);
            c.n = ic.n;
            c.by = ic.by;
            c.tb = ic.tb;
        } else {
            coords[st] = make_int4(0, 0, 0, 0);
        }
        *wcl = c;
    };
    // the (w, k) table: w = Δ·s_k·s_l, k = −2^20·w for column l and class of k
    if (threadIdx.x < 48) wktab[threadIdx.x] = make_double2(p.w[threadIdx.x], -1048576.0 * p.w[threadIdx.x]);
    if (lane == 0) {
        *wcl = WarpClaims{0, 0, 0, 0, 0, 0, 0};
        for (int st = 0; st < kUStages; ++st) mbar_init(&bars[st], 1);
        fence_mbar_init();
        prefetch_tmap(&tin);
        if (p.has_recon) prefetch_tmap(&tout);
        for (int st = 0; st < kUStages - 1; ++st) issue_next(st);
    }
    __syncthreads();   // the (w, k) table is complete

    // ---- per-lane constants (lane t is column l = t in the column passes)
    const int l = t;
    const int cl = uclass(l);
    float cq[3];          // 1/(Δ·sqrt(g_k·g_l)) per class of k (host-computed, p.cq)
    uint32_t orm[3];      // all ones where (k, l) is a rational cell (never re-checked)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        cq[c] = p.cq[l][c];
        orm[c] = c == cl ? 0xFFFFFFFFu : 0u;
    }
    const uint32_t hi_lo = kRoundHi, hi_top = kRoundHi + static_cast<uint32_t>(p.maxpix);

    unsigned long long acc = 0;
    int cur_n = -1;
    for (int it = 0;; ++it) {
        const int s = it % kUStages;
        uint8_t* stage = wbase + s * Cfg::kStageBytes;
        const int4 cd = coords[s];
        if (!cd.w) break;   // claims only grow: every later stage is empty too
        mbar_wait(&bars[s], (it / kUStages) & 1);
        TileCursor cc;
        cc.n = cd.x;
        cc.by = cd.y;
        cc.tb = cd.z;
        const int n = cc.n, by = cc.by, x0 = cc.x0();
        if (n != cur_n) {
#pragma unroll
            for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (lane == 0 && acc) flush_sse_u(sse, p, cur_n, acc);
            acc = 0;
            cur_n = n;
        }
        const int nb = min(kWTile, p.BX - x0 / 16);
        const bool row_valid = by * 16 + t < p.VH;
        uint32_t tile_sse = 0;   // <= 4 block rows x 16 x maxpix² < 2^26 per lane and tile
#pragma unroll 1
        for (int q = 0; 4 * q < nb; ++q) {
            const int bA = 4 * q + 2 * h, bB = bA + 1;
            // ---- row t of blocks A and B: Y[t][:] = X[t][:]·Tᵀ (packed)
            int aA0, aA1, aB0, aB1;
            row_addr<ELEM>(bA, t, &aA0, &aA1);
            row_addr<ELEM>(bB, t, &aB0, &aB1);
            {
                uint32_t wA[4 * ELEM], wB[4 * ELEM];
                load_px<ELEM>(stage, aA0, aA1, wA);
                load_px<ELEM>(stage, aB0, aB1, wB);
                F2 x[16], y[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) x[j] = F2{make_float2(px_f<ELEM>(wA, j), px_f<ELEM>(wB, j))};
                net_fwd(x, y);
#pragma unroll
                for (int c = 0; c < 8; ++c)
                    *reinterpret_cast<float4*>(xph + t * 128 + ((c ^ (t & 7)) << 4)) =
                        make_float4(y[2 * c].v.x, y[2 * c].v.y, y[2 * c + 1].v.x, y[2 * c + 1].v.y);
            }
            __syncwarp();
            // ---- column l: Z[:, l] = T·Y[:, l] (packed); Z of each block to the lane's buffer
            {
                F2 col[16], z[16];
#pragma unroll
                for (int k = 0; k < 16; ++k) col[k] = F2{*reinterpret_cast<const float2*>(xph + xp_off(k, l))};
                net_fwd(col, z);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    *reinterpret_cast<float4*>(zb + ((j ^ (lane & 7)) << 4)) =
                        make_float4(z[4 * j].v.x, z[4 * j + 1].v.x, z[4 * j + 2].v.x, z[4 * j + 3].v.x);
                    *reinterpret_cast<float4*>(zb + (((4 + j) ^ (lane & 7)) << 4)) =
                        make_float4(z[4 * j].v.y, z[4 * j + 1].v.y, z[4 * j + 2].v.y, z[4 * j + 3].v.y);
                }
            }
            __syncwarp();
            // ---- per block of the pair (a rolled loop: one copy of the float64 code):
            // quantiser, level -> float64 input, column inverse, transposition, row
            // inverse, rounding, SSE, reconstruction
#pragma unroll 1
            for (int half = 0; half < 2; ++half) {
                const int bb = bA + half;
                const bool valid = bb < nb;
                float zk[16];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const float4 v = *reinterpret_cast<const float4*>(zb + (((4 * half + j) ^ (lane & 7)) << 4));
                    zk[4 * j] = v.x;
                    zk[4 * j + 1] = v.y;
                    zk[4 * j + 2] = v.z;
                    zk[4 * j + 3] = v.w;
                }
                // bits = magic + m·2^F + F fraction bits, m = floor(|Z|·c + 1/2 + δ)
                uint32_t bits[16];
                uint32_t wmin = 0xFFFFFFFFu;
#pragma unroll
                for (int k = 0; k < 16; ++k) {
                    const int ck = uclass(k);
                    bits[k] = __float_as_uint(__fadd_rd(fmaf(fabsf(zk[k]), cq[ck], p.half_delta), p.magic_f));
                    wmin = min(wmin, (bits[k] & p.fmask) | orm[ck]);
                }
                double c[16];
                double2 wk[3];   // (Δ·s_k·s_l, −2^20·Δ·s_k·s_l) per class of k
#pragma unroll
                for (int cc3 = 0; cc3 < 3; ++cc3) wk[cc3] = wktab[l * 3 + cc3];
#pragma unroll
                for (int k = 0; k < 16; ++k) {
                    const int ck = uclass(k);
                    const uint32_t hi = __umulhi(bits[k], p.hi_mul) + p.hi_add;  // high word of 2^20 + m
                    const double d = __hiloint2double(static_cast<int>(hi), 0);
                    const double cm = fma(d, wk[ck].x, wk[ck].y);                // m·Δ·s_k·s_l, exact product rounded once
                    c[k] = __hiloint2double(__double2hiint(cm) ^ static_cast<int>(__float_as_uint(zk[k]) & 0x80000000u),
                                            __double2loint(cm));
                }
                if (__any_sync(0xffffffffu, wmin < p.wbits)) {
                    // irrational cell with its fraction in the window: decide exactly
#pragma unroll
                    for (int k = 0; k < 16; ++k) {
                        const int ck = uclass(k);
                        if (((bits[k] & p.fmask) | orm[ck]) < p.wbits)
                            c[k] = exact_level_input(zk[k], bits[k], p.magic_f, p.F, p.step, g_of(k) * g_of(l), wk[ck].x);
                    }
                }
                double u[16];
                net_inv(c, u);
#pragma unroll
                for (int i = 0; i < 16; ++i) *reinterpret_cast<double*>(xph + xp_off(i, l)) = u[i];
                __syncwarp();
                // ---- row i = t: A′[t][:] = (Tᵀ·B̂)[t][:]·T, rounding, SSE, reconstruction
                double rr[16], a[16];
#pragma unroll
                for (int c2 = 0; c2 < 8; ++c2) {
                    const double2 v = *reinterpret_cast<const double2*>(xph + t * 128 + ((c2 ^ (t & 7)) << 4));
                    rr[2 * c2] = v.x;
                    rr[2 * c2 + 1] = v.y;
                }
                net_inv(rr, a);
                int a0, a1;
                row_addr<ELEM>(bb, t, &a0, &a1);
                uint32_t ow[4 * ELEM];
                load_px<ELEM>(stage, a0, a1, ow);
                uint32_t lomin = 0xFFFFFFFFu, himin = 0xFFFFFFFFu, himax = 0u;
                uint32_t hiw[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const double dr = __dadd_rd(a[j], round_magic());
                    hiw[j] = static_cast<uint32_t>(__double2hiint(dr));
                    const uint32_t lo = static_cast<uint32_t>(__double2loint(dr));
                    if (j & 1) {
                        lomin = __vimin3_u32(lomin, lo, lo);
                        himin = __vimin3_u32(himin, hiw[j - 1], hiw[j]);
                        himax = __vimax3_u32(himax, hiw[j - 1], hiw[j]);
                    } else {
                        lomin = min(lomin, lo);
                    }
                }
                uint32_t e = 0;
                uint32_t out[4 * ELEM];
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    // 0x41380000 + original pixel (both have a zero low half / byte slots)
                    const uint32_t ko = ELEM == 1 ? __byte_perm(ow[j >> 2], kRoundHi, 0x7650 | (j & 3))
                                                  : __byte_perm(ow[j >> 1], kRoundHi, (j & 1) ? 0x7632 : 0x7610);
                    const int dd = static_cast<int>(hiw[j] - ko);
                    e += static_cast<uint32_t>(dd * dd);
                }
                if (ELEM == 1) {
#pragma unroll
                    for (int q4 = 0; q4 < 4; ++q4)
                        out[q4] = __byte_perm(__byte_perm(hiw[4 * q4], hiw[4 * q4 + 1], 0x0040),
                                              __byte_perm(hiw[4 * q4 + 2], hiw[4 * q4 + 3], 0x0040), 0x5410);
                } else {
#pragma unroll
                    for (int q2 = 0; q2 < 8; ++q2) out[q2] = __byte_perm(hiw[2 * q2], hiw[2 * q2 + 1], 0x5410);
                }
                // lo < 2^13: within 2^-20 of a .5 boundary; hi outside [K, K + maxpix]: clamp
                const bool slow = valid && (lomin < 8192u || himin < hi_lo || himax > hi_top);
                if (__any_sync(0xffffffffu, slow)) {
                    if (slow) {
                        uint32_t o2[4 * ELEM], r2[4 * ELEM];   // local copies: the call takes addresses
#pragma unroll
                        for (int q2 = 0; q2 < 4 * ELEM; ++q2) o2[q2] = ow[q2];
                        double row[16];
                        for (int j = 0; j < 16; ++j) row[j] = *reinterpret_cast<const double*>(xph + xp_off(t, j));
                        e = exact_row<ELEM>(stage, bb, row, t, p.step, p.maxpix, o2, r2);
#pragma unroll
                        for (int q2 = 0; q2 < 4 * ELEM; ++q2) out[q2] = r2[q2];
                    }
                    // the exact branch re-reads the block's ORIGINAL pixels: no lane may
                    // write its reconstructed row before every lane is past it
                    __syncwarp();
                }
                if (valid && row_valid) tile_sse += e;
                if (p.has_recon) {
                    *reinterpret_cast<uint4*>(stage + a0) = make_uint4(out[0], out[1], out[2], out[3]);
                    if (ELEM == 2) *reinterpret_cast<uint4*>(stage + a1) = make_uint4(out[4], out[5], out[6], out[7]);
                }
                __syncwarp();   // the transposition tile is rewritten next
            }
        }
        acc += tile_sse;
        if (lane == 0) {
            if (p.has_recon) {
                fence_async_smem();
                w_store_at<ELEM>(&tout, p, cc, stage);
                bulk_commit();
                bulk_wait_read<1>();   // the store of the previous tile has left the stage refilled next
            }
            issue_next((it + kUStages - 1) % kUStages);
        }
        __syncwarp();
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
        if (acc) flush_sse_u(sse, p, cur_n, acc);
        if (p.has_recon) bulk_wait<0>();
        claims_done(sched, p.total_warps);
    }
}


namespace {

template <int ELEM>
int launch_cu(const void* src, const Geom& g, const dct16a_quant& q, void* recon, uint64_t* sse, cudaStream_t st,
              uint64_t* const* peers, int n_peers, long long frame_offset, int multicast) {
    using Cfg = UCfg<ELEM>;
    CUtensorMap tin, tout;
    const uint64_t dims[3] = {uint64_t(g.W), uint64_t(g.H), uint64_t(g.N)};
    const uint64_t strides[2] = {uint64_t(g.pitch), uint64_t(g.istride)};
    const uint32_t box[3] = {uint32_t(128 / ELEM), 16u, 1u};
    const CUtensorMapDataType dt = ELEM == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_UINT16;
    if (encode_tiled(&tin, dt, 3, src, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B,
                     ELEM == 1 ? CU_TENSOR_MAP_L2_PROMOTION_NONE : CU_TENSOR_MAP_L2_PROMOTION_L2_256B))
        return DCT16A_ECUDA;
    if (recon) {
        if (encode_tiled(&tout, dt, 3, recon, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_NONE))
            return DCT16A_ECUDA;
    } else {
        tout = tin;
    }
    UParams p{};
    p.W = g.W;
    p.BX = g.BX;
    p.BY = g.BY;
    p.VH = g.VH;
    p.tiles_per_strip = (g.BX + kWTile - 1) / kWTile;
    p.maxpix = (1 << g.bits) - 1;
    p.n_tiles = static_cast<long long>(g.N) * g.BY * p.tiles_per_strip;
    p.has_recon = recon != nullptr;
    p.n_peers = n_peers;
    p.multicast = multicast;
    p.frame_offset = frame_offset;
    for (int i = 0; i < n_peers; ++i) p.peers[i] = reinterpret_cast<unsigned long long*>(peers[i]);
    p.step = q.step;
    // e = |Z|/(Δ·sqrt(G)) + 1/2 <= e_max; its float error is <= e_max·2^-23 (the
    // rounded constant and the fma); δ = 2·err keeps the rational cells exact
    // because δ + err < 1/(32Δ), the smallest spacing of their e (reading A9).
    const double e_max = 16.0 * p.maxpix / q.step + 1.0;
    const double err = e_max * 0x1p-23;
    int nbits = 0;
    while ((1 << nbits) <= static_cast<int>(e_max) + 1) ++nbits;
    p.F = 22 - nbits;                     // m < 2^nbits below the magic's 1.5
    p.fmask = (1u << p.F) - 1u;
    const float hd = static_cast<float>(0.5 + 2.0 * err);
    const double delta = static_cast<double>(hd) - 0.5;
    if (!(delta > err && delta + err < 1.0 / (32.0 * q.step))) return DCT16A_EDOMAIN;
    p.half_delta = hd;
    p.magic_f = 1.5f * static_cast<float>(1 << (23 - p.F));
    uint32_t magic_bits;
    memcpy(&magic_bits, &p.magic_f, 4);
    p.wbits = static_cast<uint32_t>(ceil((delta + 2.0 * err) * (1 << p.F)));
    // high word of the double 2^20 + m (m < 2^19): 0x41300000 + m = (bits >> F) - (magic_bits >> F) + 0x41300000
    p.hi_mul = 1u << (32 - p.F);
    p.hi_add = 0x41300000u - (magic_bits >> p.F);
    for (int l = 0; l < 16; ++l)
        for (int c = 0; c < 3; ++c) {
            const int kk = c == 0 ? 0 : (c == 1 ? 2 : 3);   // representatives of g = 16, 12, 8
            const double s = s_of(kk) * s_of(l);
            p.cq[l][c] = static_cast<float>(s / q.step);
            p.w[3 * l + c] = static_cast<double>(q.step) * s;
        }
    if (int e = smem_optin(reinterpret_cast<const void*>(codec_uniform_kernel<ELEM>), Cfg::kSmem)) return e;
    long long grid = static_cast<long long>(num_sms()) * Cfg::kCtasPerSm;
    p.claim = static_cast<int>(std::min<long long>(kUClaim, std::max<long long>(1, p.n_tiles / (grid * kUWarps * 4))));
    const long long want = (p.n_tiles + kUWarps * p.claim - 1) / (kUWarps * p.claim);
    if (want < grid) grid = want;
    p.total_warps = static_cast<int>(grid) * kUWarps;
    SchedGuard guard(kSchedCodecUniform, st);
    if (guard.error()) return guard.error();
    p.slot = guard.slot();
    codec_uniform_kernel<ELEM><<<static_cast<unsigned>(grid), kUWarps * 32, Cfg::kSmem, st>>>(
        tin, tout, reinterpret_cast<unsigned long long*>(sse), p);
    return static_cast<int>(cudaGetLastError());
}

}  // namespace

int launch_codec_uniform(const void* src, const Geom& g, const dct16a_quant& q, void* recon, uint64_t* sse,
                         cudaStream_t st, uint64_t* const* peers, int n_peers, long long frame_offset, int multicast) {
    if (g.elem == 1) return launch_cu<1>(src, g, q, recon, sse, st, peers, n_peers, frame_offset, multicast);
    return launch_cu<2>(src, g, q, recon, sse, st, peers, n_peers, frame_offset, multicast);
}

}  // namespace dct16a
#endif  // DCT16A_EXPERIMENTS
