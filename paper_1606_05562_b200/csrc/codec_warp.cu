// codec_warp.cu — the fused codec with 16 lanes per 16x16 block (one warp holds
// a block pair): forward, quantisation with S folded in
// (PAPER.md:305-344), inverse (896-901), round half away / clamp (reading A6),
// per-image SSE (906-910).  It serves the uniform quantiser (config 4, any bit
// depth), the zonal cases the band kernel does not cover (r > 136) and, with
// DCT16A_OPT_CODEC_PATH = 2, every zonal case (the GPU tests cross-check it
// against the band kernel).
//
// * Data: each warp streams tiles of 8 blocks (16 rows x 128 px) through a
//   3-stage TMA ring in the 128-byte swizzle, so the lanes of a quarter-warp
//   (rows 0-7 of one block) read distinct 16-byte chunks with ld.shared.v4;
//   the reconstruction overwrites the tile in place and leaves by TMA store.
// * Forward: lane t holds row t, the row pass runs the 60-add network of
//   Eq. (1) in float32 (exact: every partial sum is an integer < 2^24, V9);
//   the transposition buffer of the paper is a per-warp
//   smem tile; lane l then runs the column pass on column l.
// * Uniform quantiser (reading A9): m = floor(|Z|·c + 1/2 + δ) from one FMA and
//   one round-down magic add keeping F fraction bits.  δ (> the float error,
//   below the 1/(2Δ·sqrt(G)) spacing of the rational cells) makes the rational
//   cells — the only ones with exact ties — exact; in the irrational cells a
//   value whose fraction falls in the window [0, δ + 2·err) is re-decided
//   exactly in integers (uniform_fix).
// * Uniform inverse in float64 (reading A10): the level enters as the double
//   1.5·2^E + m whose high word is one IMAD of the float's bits; one DFMA with
//   the weight Δ·s_k·s_l and the constant −fl(1.5·2^E·w) forms the input
//   (error < 1e-11) and the sign of Z flips the result's sign bit; two 60-add
//   networks, smem transposition in between; rounding by one round-down add
//   onto 1.5·2^20 + 1/2 (high word = pixel, low word = fraction), clamp by one
//   relu-min; a pixel within 2^-20 of a .5 boundary sends the warp to the exact
//   decision (uexact_tile.cuh: block_levels_coop → block_components_coop →
//   exact_row_fix_levels).
// * Zonal inverse in float32, exact (half-integers < 2^23): N + 1152.5 on the
//   DC input, pixel = floor((N + 1152.5)/2304) by one round-down FMA; 8-bit
//   pixels are clamped and packed by cvt.pack.sat.
// * SSE: per row, vabsdiff4/dp4a (8-bit) or integer squares (10-bit), one
//   64-bit atomic per warp and image (or, for dct16a_codec_allreduce, into
//   every rank's vector over peer memory).
// * Schedule: persistent warps claim runs of consecutive tiles from a global
//   counter (dynamic scheduler, compact address window) and walk each run with
//   an incremental tile cursor (tile128.cuh).
#include <cuda.h>
#include <stdint.h>
#include <math.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <type_traits>

#include "internal.h"
#include "net16.cuh"
#include "ptx.cuh"
#include "sched.cuh"
#include "quant.cuh"
#include "tables.cuh"
#include "tile128.cuh"
#include "uexact.cuh"
#include "uexact_tile.cuh"

namespace dct16a {
namespace {

#ifndef DCT16A_CW_PROMO
#define DCT16A_CW_PROMO 3   // input L2 promotion (CUtensorMapL2promotion): 256 B
#endif
#ifndef DCT16A_CW_STAGES
#define DCT16A_CW_STAGES 3
#endif
#ifndef DCT16A_CW_UCTAS
#define DCT16A_CW_UCTAS 3
#endif
constexpr int kWWarps = 4;                  // warps per CTA
constexpr int kWStages = DCT16A_CW_STAGES;  // TMA ring depth per warp
// per-warp transposition bytes (2 blocks x 16 x 17 doubles = 4352), rounded so
// that every warp's stages stay 1024-byte aligned (the 128-byte swizzle pattern
// is taken from smem address bits 7-9)
constexpr int kWXpose = 5120;

template <int ELEM, bool UNIFORM>
struct WCfg {
    static constexpr int kStageBytes = 16 * kWTile * 16 * ELEM;   // 2 KB (u8) / 4 KB (u16)
    static constexpr int kWarpBytes = kWStages * kStageBytes + kWXpose;
    static_assert(kWarpBytes % 1024 == 0, "stages must stay 1024-byte aligned");
    // + per warp: kWStages mbarriers and the coordinates (n, by, tb, valid) of each stage's tile
    static constexpr int kSmem = 1024 + kWWarps * kWarpBytes + kWWarps * kWStages * (8 + 16);
    static constexpr int kFit = (227 * 1024) / (kSmem + 1024);
    // the float64 path needs ~170 registers: at most 3 CTAs (12 warps) per SM
    static constexpr int kCtasPerSm = UNIFORM ? (kFit < DCT16A_CW_UCTAS ? kFit : DCT16A_CW_UCTAS) : (kFit < 4 ? kFit : 4);
};

constexpr int kMaxPeers = 8;

#ifndef DCT16A_CW_CLAIM
#define DCT16A_CW_CLAIM 4
#endif
constexpr int kWClaim = DCT16A_CW_CLAIM;   // consecutive tiles per claim
// Dynamic tile scheduler (sched.cuh, as in forward.cu / zonal_band.cu): runs of
// kWClaim tiles claimed in increasing order from a global counter keep the
// tiles in flight in one compact address window.
__device__ unsigned long long g_cw_sched[kSchedSlots][2];

struct WParams {
    int W, BX, BY, VH, tiles_per_strip, maxpix;
    long long n_tiles;
    int slot, total_warps, claim;   // tile scheduler (sched.cuh; slot -1 = static), tiles per claim
    int has_recon;
    // fused SSE all-reduce (dct16a_codec_allreduce): every image's SSE is added
    // into sse_peers[q][frame_offset + n] of every peer q; n_peers = 0: local sse
    int n_peers, multicast;   // multicast: peers[0] is an NVLS multicast address
    long long frame_offset;
    unsigned long long* peers[kMaxPeers];
    // zonal
    int r;
    // uniform
    int step, F, wbits, hi_shift, hi_c, hi_c2;
    uint32_t hi_mult;   // 2^hi_shift (an opaque multiplier: one IMAD builds the high word)
    float magic_f, half_delta;
    uint32_t magic_bits;
    // uniform, fixed-point quantiser (intq = 1): e·2^32 = |Z|·C + H exactly in 64 bits,
    // C = round(2^32/(Δ·sqrt(G))) per cell class, H = (1/2 + δ)·2^32; window wlo
    int intq;
    uint32_t wlo, hfix;   // hfix < 2^32
};

// |Z| of an integer-valued float (|Z| < 2^23) as an integer: the product with
// 2^-149 is the subnormal whose bit pattern is |Z| (exact; denormals are kept:
// the library is built without flush-to-zero, tests/test_abi.py checks it).
__device__ __forceinline__ uint32_t abs_z_bits(float z) { return __float_as_uint(__fmul_rn(fabsf(z), 0x1p-149f)); }

// |Z|·C + H in 64 bits by one IMAD.WIDE.U32 (inline PTX: the compiler would
// otherwise split the add of H off the multiply); returns the low word, *hi = the high word.
__device__ __forceinline__ uint32_t mad_wide_u32(uint32_t a, uint32_t b, unsigned long long c, uint32_t* hi) {
    unsigned long long e;
    asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(e) : "r"(a), "r"(b), "l"(c));
    uint32_t lo, h;
    asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(h) : "l"(e));
    *hi = h;
    return lo;
}

// Exact uniform level for a coefficient whose float estimate m is flagged (rare).
__device__ __noinline__ int32_t uniform_fix_call(float z, int32_t m, int step, int G) {
    const uint32_t az = static_cast<uint32_t>(fabsf(z));
    return uniform_fix(az, m, static_cast<uint64_t>(step) * step * G);
}

// The rare re-decision of a lane's flagged coefficients (bit k of `flagged`: the
// fraction of coefficient k's level estimate lies in the window), kept compact
// for the instruction cache: a rolled loop over the flagged k only, the exact
// level by uniform_fix (from a float estimate; it corrects by one step), the
// new input of the float64 inverse into a per-lane slot of the warp's
// transposition tile (free between the column pass and the inverse), then the
// flagged registers reloaded.  The whole warp calls it (it synchronises).
__device__ __forceinline__ void refix_levels(uint32_t flagged, const float (&z)[16], double (&c)[16], uint8_t* xpose,
                                          int lane, const float (&cq)[3], const double (&wq)[3],
                                          const double (&kq)[3], int l, const WParams& p) {
    double* slot = reinterpret_cast<double*>(xpose) + lane * 16;
    const int gl = g_of(l);
    for (uint32_t f = flagged; f; f &= f - 1) {
        const int k = __ffs(f) - 1;
        float zk = 0.0f;
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) zk = kk == k ? z[kk] : zk;
        const int ck = uclass(k);
        const float cqk = ck == 0 ? cq[0] : (ck == 1 ? cq[1] : cq[2]);
        const double wqk = ck == 0 ? wq[0] : (ck == 1 ? wq[1] : wq[2]);
        const double kqk = ck == 0 ? kq[0] : (ck == 1 ? kq[1] : kq[2]);
        const uint32_t az = static_cast<uint32_t>(fabsf(zk));
        const int32_t m0 = static_cast<int32_t>(fmaf(static_cast<float>(az), cqk, 0.5f));   // within one of the level
        const int32_t m = uniform_fix(az, m0, static_cast<uint64_t>(p.step) * p.step * (g_of(k) * gl));
        const double cm = fma(__hiloint2double((m << p.hi_shift) + p.hi_c, 0), wqk, kqk);
        slot[k] = zk < 0.0f ? -cm : cm;
    }
#pragma unroll
    for (int k = 0; k < 16; ++k)
        if (flagged & (1u << k)) c[k] = slot[k];
    __syncwarp();   // the slots are the transposition tile the inverse writes next
}

}  // namespace

// Add one image's SSE: locally, or into every rank's vector — with one
// multimem.red on the NVLS multicast address (the NVSwitch applies the add to
// every GPU's copy) or with system-scope 64-bit atomics on each peer-mapped
// vector over NVLink.  Integer adds are order-independent, so every rank ends
// with the exact per-frame sums: the path's all-reduce.
__device__ __forceinline__ void flush_sse(unsigned long long* sse, const WParams& p, int n, unsigned long long v) {
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

// FIXQ: the uniform quantiser in 64-bit fixed point (steps small enough for its
// error bound, launch_cw); otherwise in float32
template <int ELEM, bool UNIFORM, bool FIXQ = false>
__global__ void __launch_bounds__(kWWarps * 32, WCfg<ELEM, UNIFORM>::kCtasPerSm)
    codec_warp_kernel(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout,
                      unsigned long long* __restrict__ sse, const WParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = walign1024(smem_raw);
    using Cfg = WCfg<ELEM, UNIFORM>;
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int h = lane >> 4, t = lane & 15;
    uint8_t* wbase = smem + warp * Cfg::kWarpBytes;
    uint8_t* xpose = wbase + kWStages * Cfg::kStageBytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kWWarps * Cfg::kWarpBytes) + warp * kWStages;

    int4* coords = reinterpret_cast<int4*>(smem + kWWarps * Cfg::kWarpBytes + kWWarps * kWStages * 8) +
                   warp * kWStages;
    const uint64_t pol = policy_evict_first();
    unsigned long long* sched = p.slot >= 0 ? g_cw_sched[p.slot] : nullptr;
    Claims claims(sched, static_cast<long long>(blockIdx.x) * kWWarps + warp, static_cast<long long>(gridDim.x) * kWWarps);   // lane 0

    // lane 0: the claim in progress (tiles [next, end)) and its cursor
    long long next = 0, end = 0;
    TileCursor ic;
    auto issue_next = [&](int st) {   // claim the next tile, load it into stage st (lane 0)
        if (next == end) {
            const long long first = claims.next() * p.claim;
            next = first;
            end = first < p.n_tiles ? min(first + p.claim, p.n_tiles) : first;
            if (first < p.n_tiles) ic.init(p, first);
        }
        if (next < end) {
            coords[st] = make_int4(ic.n, ic.by, ic.tb, 1);
            w_issue_at<ELEM>(&tin, p, ic, wbase + st * Cfg::kStageBytes, &bars[st], pol);
            ++next;
            ic.advance(p);
        } else {
            coords[st] = make_int4(0, 0, 0, 0);
        }
    };
    if (lane == 0) {
        for (int st = 0; st < kWStages; ++st) mbar_init(&bars[st], 1);
        fence_mbar_init();
        prefetch_tmap(&tin);
        if (p.has_recon) prefetch_tmap(&tout);
        for (int st = 0; st < kWStages - 1; ++st) issue_next(st);
    }
    __syncwarp();

    // ---- per-lane constants (lane t is column l = t in the column pass)
    const int l = t;
    const int cl = uclass(l);
    float cq[3];          // uniform: 1/(Δ·sqrt(g_k·g_l)) per class of k
    double wq[3], kq[3];  // uniform: Δ·s_k·s_l and −fl(1.5·2^E·Δ·s_k·s_l)
    uint32_t orm[3];      // uniform: all ones where the cell (k, l) is rational (never re-checked)
    uint32_t cfix[3];     // uniform, fixed point: round(2^32/(Δ·sqrt(g_k·g_l))) per class of k
    float wz[16];         // zonal: W ⊙ M_r
    if constexpr (UNIFORM) {
        const double sl = s_of(l);
        const double Kmag = static_cast<double>(3LL << (19 - p.hi_shift));   // 1.5·2^E, E = 20 - hi_shift
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const int kk = c == 0 ? 0 : (c == 1 ? 2 : 3);   // representatives of g = 16, 12, 8
            const double s = s_of(kk) * sl;
            cq[c] = static_cast<float>(s / p.step);
            cfix[c] = static_cast<uint32_t>(__double2ull_rn(ldexp(s / p.step, 32)));
            wq[c] = static_cast<double>(p.step) * s;
            kq[c] = -(Kmag * wq[c]);
            orm[c] = c == cl ? 0xFFFFFFFFu : 0u;
        }
    } else {
#pragma unroll
        for (int k = 0; k < 16; ++k) wz[k] = zigzag_rank(k, l) < p.r ? static_cast<float>(w_of(k, l)) : 0.0f;
    }
    const uint32_t fmask = (1u << p.F) - 1u;

    // per-warp transposition tiles: Y (float, row pitch 20, second block shifted 16 banks)
    // and U (V = double, row pitch 18: 144-byte rows, so a row is read with 16-byte
    // loads and every quarter-warp phase of them hits distinct banks; float: pitch 17)
    float* ty = reinterpret_cast<float*>(xpose) + h * (16 * 20 + 16);
    using V = typename std::conditional<UNIFORM, double, float>::type;
    constexpr int kTuP = UNIFORM ? 18 : 17;
    V* tu = reinterpret_cast<V*>(xpose) + h * (16 * kTuP);

    unsigned long long acc = 0;
    int cur_n = -1;
    for (int it = 0;; ++it) {
        const int s = it % kWStages;
        uint8_t* stage = wbase + s * Cfg::kStageBytes;
        const int4 cd = coords[s];
        if (!cd.w) break;   // claims only grow: every later stage is empty too
        mbar_wait(&bars[s], (it / kWStages) & 1);
        TileCursor cc;
        cc.n = cd.x;
        cc.by = cd.y;
        cc.tb = cd.z;
        const int n = cc.n, by = cc.by, x0 = cc.x0();
        if (n != cur_n) {
#pragma unroll
            for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (lane == 0 && acc) flush_sse(sse, p, cur_n, acc);
            acc = 0;
            cur_n = n;
        }
        const int nb = min(kWTile, p.BX - x0 / 16);
        const bool row_valid = by * 16 + t < p.VH;
#pragma unroll 1
        for (int pair = 0; 2 * pair < nb; ++pair) {
            const int bb = 2 * pair + h;
            const bool valid = bb < nb;
            int a0, a1;
            row_addr<ELEM>(bb, t, &a0, &a1);
            // ---- row t: Y[t][:] = X[t][:]·Tᵀ
            {
                uint32_t w[4 * ELEM];
                load_px<ELEM>(stage, a0, a1, w);
                float x[16], y[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) x[j] = px_float<ELEM>(w, j);
                net_fwd(x, y);
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    *reinterpret_cast<float4*>(ty + t * 20 + 4 * q) = make_float4(y[4 * q], y[4 * q + 1], y[4 * q + 2], y[4 * q + 3]);
            }
            __syncwarp();
            // ---- column l: Z[:, l] = T·Y[:, l]
            float z[16];
            {
                float col[16];
#pragma unroll
                for (int k = 0; k < 16; ++k) col[k] = ty[k * 20 + l];
                net_fwd(col, z);
            }
            __syncwarp();
            // ---- quantise, weight, inverse down the column
            {
                V c[16], u[16];
                if constexpr (UNIFORM) {
                    // level m = floor(e), e = |Z|·c + 1/2 + δ.  δ (> the evaluation error,
                    // below the 1/(32Δ) spacing of the rational cells) makes the rational
                    // cells — the only ones with exact ties — exact; an irrational cell whose
                    // fraction falls in the window [0, δ + 2·err) is re-decided in integers.
                    // The level enters the float64 inverse as the double 1.5·2^E + m (its
                    // high word one IMAD of m) times the weight by one DFMA; the sign of Z
                    // flips the result's sign bit.
                    uint32_t nmin = 0xFFFFFFFFu;
                    if constexpr (FIXQ) {
                        const unsigned long long hfix64 = p.hfix;
                        // fixed point: |Z|·C + H = (e + error)·2^32 exactly in 64 bits (one
                        // IMAD.WIDE), C = round(2^32·c), H = (1/2 + δ)·2^32: m is the high
                        // word, the fraction the low word
#pragma unroll
                        for (int k = 0; k < 16; ++k) {
                            const int ck = uclass(k);
                            const uint32_t az = abs_z_bits(z[k]);
                            uint32_t m;
                            const uint32_t fr = mad_wide_u32(az, cfix[ck], hfix64, &m);
                            nmin = min(nmin, fr | orm[ck]);
                            const double d = __hiloint2double(static_cast<int>(m * p.hi_mult + p.hi_c), 0);
                            const double cm = fma(d, wq[ck], kq[ck]);
                            c[k] = __hiloint2double(__double2hiint(cm) ^ static_cast<int>(__float_as_uint(z[k]) & 0x80000000u),
                                                    __double2loint(cm));
                        }
                        if (__any_sync(0xffffffffu, nmin < p.wlo)) {
                            uint32_t flagged = 0;
#pragma unroll
                            for (int k = 0; k < 16; ++k) {
                                uint32_t m0;
                                const uint32_t fr = mad_wide_u32(abs_z_bits(z[k]), cfix[uclass(k)], hfix64, &m0);
                                if ((fr | orm[uclass(k)]) < p.wlo) flagged |= 1u << k;
                            }
                            refix_levels(flagged, z, c, xpose, lane, cq, wq, kq, l, p);
                        }
                    } else {
                        // float32 (steps too large for the fixed point's error bound): one FMA
                        // and one round-down magic add onto 1.5·2^(23-F) keeping F fraction bits
#pragma unroll
                        for (int k = 0; k < 16; ++k) {
                            const int ck = uclass(k);
                            const float e = fmaf(fabsf(z[k]), cq[ck], p.half_delta);
                            const uint32_t bits = __float_as_uint(__fadd_rd(e, p.magic_f));
                            nmin = min(nmin, (bits & fmask) | orm[ck]);
                            const double d = __hiloint2double(static_cast<int>((bits >> p.F) * p.hi_mult + p.hi_c2), 0);
                            const double cm = fma(d, wq[ck], kq[ck]);
                            c[k] = __hiloint2double(__double2hiint(cm) ^ static_cast<int>(__float_as_uint(z[k]) & 0x80000000u),
                                                    __double2loint(cm));
                        }
                        // irrational cell with its fraction in the window [0, δ + 2·err): decide exactly
                        if (__any_sync(0xffffffffu, nmin < static_cast<uint32_t>(p.wbits))) {
                            uint32_t flagged = 0;   // the lane's coefficients in the window
#pragma unroll
                            for (int k = 0; k < 16; ++k) {
                                const float e = fmaf(fabsf(z[k]), cq[uclass(k)], p.half_delta);
                                const uint32_t bits = __float_as_uint(__fadd_rd(e, p.magic_f));
                                if (((bits & fmask) | orm[uclass(k)]) < static_cast<uint32_t>(p.wbits)) flagged |= 1u << k;
                            }
                            refix_levels(flagged, z, c, xpose, lane, cq, wq, kq, l, p);
                        }
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < 16; ++k) c[k] = z[k] * wz[k];
                    if (l == 0) c[0] += 1152.5f;   // N + 1152.5 everywhere: rounding offset on the DC input
                }
                net_inv(c, u);
#pragma unroll
                for (int i = 0; i < 16; ++i) tu[i * kTuP + l] = u[i];
            }
            __syncwarp();
            // ---- row i = t: A′[i][:] = (Tᵀ·B̂)[i][:]·T, round, clamp
            int pix[16];
            {
                V rr[16], a[16];
                if constexpr (UNIFORM) {
#pragma unroll
                    for (int j = 0; j < 16; j += 2) {
                        const double2 v2 = *reinterpret_cast<const double2*>(tu + t * kTuP + j);
                        rr[j] = v2.x;
                        rr[j + 1] = v2.y;
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 16; ++j) rr[j] = tu[t * kTuP + j];
                }
                net_inv(rr, a);
                if constexpr (UNIFORM) {
                    // floor(A′ + 1/2) from one round-down add (round_f64); any pixel within
                    // 2^-20 of a .5 boundary sends the warp to the exact decision
                    uint32_t nmin = 0xFFFFFFFFu;
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const double d = __dadd_rd(a[j], 1572864.5);
                        nmin = min(nmin, static_cast<uint32_t>(__double2loint(d)) + 4096u);
                        pix[j] = __vimin_s32_relu(__double2hiint(d) - 0x41380000, p.maxpix);
                    }
                    if (!valid) nmin = 0xFFFFFFFFu;
                    if (__any_sync(0xffffffffu, nmin < 8192u)) {
                        // the row's float64 values, from the transposition tile before the
                        // level computation below reuses it (local memory: rare branch only)
                        double arow[16];
                        if (nmin < 8192u) {
                            double rin[16];
                            for (int j = 0; j < 16; ++j) rin[j] = tu[t * kTuP + j];
                            net_inv(rin, arow);
                        }
                        __syncwarp();
                        // the exact levels of both blocks of the pair, computed once by their
                        // lanes from the ORIGINAL pixels (no lane has written its
                        // reconstruction yet), then — when a block with levels in
                        // irrational cells has a pixel to decide — the four integer
                        // components of every row (scratch: this half's 2.5 KB of the tile)
                        int32_t* qs = reinterpret_cast<int32_t*>(xpose) + h * 640;
                        const bool irr = block_levels_coop<ELEM>(stage, bb, t, p.step, qs);
                        const bool rational = ((__ballot_sync(0xffffffffu, irr) >> (16 * h)) & 0xFFFFu) == 0;
                        int32_t J[4][16];
                        if (__any_sync(0xffffffffu, nmin < 8192u && !rational))
                            block_components_coop(qs, qs + 320, t, J);
                        if (nmin < 8192u) {
                            int fix[16];
#pragma unroll
                            for (int j = 0; j < 16; ++j) fix[j] = pix[j];
                            exact_row_fix_levels(arow, J, rational, p.step, p.maxpix, fix);
#pragma unroll
                            for (int j = 0; j < 16; ++j) pix[j] = fix[j];
                        }
                        // the tile is rewritten next, and the levels were read from the
                        // ORIGINAL pixels: no lane may write its reconstruction before
                        __syncwarp();
                    }
                } else {
                    // floor((N + 1152.5)/2304) by one round-down FMA onto 2^23 (exact: the
                    // product errs by < 2^-24·t, below the 1/4608 distance of an odd
                    // multiple of 1/4608 to an integer for t < 3640); 8-bit clamps in the
                    // saturating pack below, 10-bit here
                    const float inv2304 = 1.0f / 2304.0f;
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const int v = static_cast<int>(__float_as_uint(__fmaf_rd(a[j], inv2304, 8388608.0f)) - 0x4B000000u);
                        pix[j] = ELEM == 1 ? v : __vimin_s32_relu(v, p.maxpix);
                    }
                }
            }
            // ---- SSE against the original row, in-place reconstruction
            {
                uint32_t w[4 * ELEM];
                load_px<ELEM>(stage, a0, a1, w);
                uint32_t e = 0;
                uint32_t o[4 * ELEM];
                if (ELEM == 1) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        // clamp to [0, 255] and pack four pixels (cvt.pack.sat)
                        o[q] = pack2_sat_u8(pix[4 * q + 1], pix[4 * q], pack2_sat_u8(pix[4 * q + 3], pix[4 * q + 2], 0u));
                        const uint32_t d = __vabsdiffu4(o[q], w[q]);
                        e = __dp4a(d, d, e);
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        o[q] = __byte_perm(pix[2 * q], pix[2 * q + 1], 0x5410);
                        const int d0 = pix[2 * q] - static_cast<int>(w[q] & 0xFFFFu);
                        const int d1 = pix[2 * q + 1] - static_cast<int>(w[q] >> 16);
                        e += static_cast<uint32_t>(d0 * d0 + d1 * d1);
                    }
                }
                if (valid && row_valid) acc += e;
                if (p.has_recon) {
                    *reinterpret_cast<uint4*>(stage + a0) = make_uint4(o[0], o[1], o[2], o[3]);
                    if (ELEM == 2) *reinterpret_cast<uint4*>(stage + a1) = make_uint4(o[4], o[5], o[6], o[7]);
                }
            }
            __syncwarp();
        }
        if (lane == 0) {
            if (p.has_recon) {
                fence_async_smem();
                w_store_at<ELEM>(&tout, p, cc, stage);
                bulk_commit();
                bulk_wait_read<1>();   // the store of tile tix-1 has left the stage refilled next
            }
            issue_next((it + kWStages - 1) % kWStages);
        }
        __syncwarp();
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
        if (acc) flush_sse(sse, p, cur_n, acc);
        if (p.has_recon) bulk_wait<0>();
        claims_done(sched, p.total_warps);   // every warp has claimed past the end
    }
}

namespace {

template <int ELEM, bool UNIFORM>
int launch_cw(const void* src, const Geom& g, const dct16a_quant& q, void* recon, uint64_t* sse, cudaStream_t st,
              uint64_t* const* peers = nullptr, int n_peers = 0, long long frame_offset = 0, int multicast = 0) {
    using Cfg = WCfg<ELEM, UNIFORM>;
    CUtensorMap tin, tout;
    const uint64_t dims[3] = {uint64_t(g.W), uint64_t(g.H), uint64_t(g.N)};
    const uint64_t strides[2] = {uint64_t(g.pitch), uint64_t(g.istride)};
    const uint32_t box[3] = {uint32_t(128 / ELEM), 16u, 1u};
    const CUtensorMapDataType dt = ELEM == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_UINT16;
    if (encode_tiled(&tin, dt, 3, src, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B,
                     static_cast<CUtensorMapL2promotion>(DCT16A_CW_PROMO)))
        return DCT16A_ECUDA;
    if (recon) {
        if (encode_tiled(&tout, dt, 3, recon, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_NONE))
            return DCT16A_ECUDA;
    } else {
        tout = tin;
    }
    WParams p{};
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
    p.r = q.r;
    p.step = q.step;
    if (UNIFORM) {
        // e = |Z|/(Δ·sqrt(G)) + 1/2 <= e_max (|Z| <= maxpix·g_k·g_l); the float
        // evaluation e' = e + δ + ε has |ε| <= err = e_max·2^-23 (the rounded c and
        // the fma).  With δ > err, e' > e, so a rational cell's exact tie (e an
        // integer) rounds up as it must and, because δ + err < 1/(32Δ) (the
        // smallest spacing of their e, reading A9), no other rational value crosses
        // an integer; an irrational cell's level is one too high only when the
        // fraction of e' is below δ + err: the window (δ = 1.25·err).
        const double e_max = 16.0 * p.maxpix / q.step + 1.0;
        const double err = e_max * 0x1p-23;
        int nbits = 0;
        while ((1 << nbits) <= static_cast<int>(e_max) + 1) ++nbits;
        p.F = 22 - nbits;
        const float hd = static_cast<float>(0.5 + 1.25 * err);
        const double delta = static_cast<double>(hd) - 0.5;
        if (!(delta > err && delta + err < 1.0 / (32.0 * q.step))) return DCT16A_EDOMAIN;
        p.half_delta = hd;
        p.magic_f = 1.5f * static_cast<float>(1 << (23 - p.F));
        memcpy(&p.magic_bits, &p.magic_f, 4);
        p.wbits = static_cast<int>(ceil((delta + err) * (1 << p.F)));
        // level -> double 1.5·2^E + m: E with 2^E > 2·m_max, m placed at bit (20 - E) of the high word
        int E = 1;
        while ((1 << E) <= 2 * (static_cast<int>(e_max) + 1)) ++E;
        p.hi_shift = 20 - E;
        p.hi_mult = 1u << p.hi_shift;
        p.hi_c = 0x3FF00000 + ((E) << 20) + (1 << 19);   // high word of 1.5·2^E
        // the same word from bits >> F = (magic_bits >> F) + m (arithmetic mod 2^32)
        p.hi_c2 = static_cast<int>(static_cast<uint32_t>(p.hi_c) - ((p.magic_bits >> p.F) << p.hi_shift));
        // fixed point: C = round(2^32·c) from a double within 2^-20 of 2^32·c, so |C − 2^32·c| <= 0.501 and
        // |Z|·C + H = (e + ε)·2^32 with |ε| <= err_fx; usable while δ > err_fx and δ + err_fx < 1/(32Δ)
        const double az_max = 256.0 * p.maxpix;
        const double err_fx = (az_max * 0.501 + 1.0) * 0x1p-32;
        const unsigned long long H = static_cast<unsigned long long>(llround(ldexp(0.5 + 1.25 * err_fx, 32)));
        const double dfx = ldexp(static_cast<double>(H), -32) - 0.5;
        const double wlo = ceil(ldexp(dfx + err_fx, 32));
        // automatic choice: fixed point for steps <= 8, where the float window flags
        // many coefficients (Δ = 1..8: 4.0-5.0 ms float against 4.04-4.08 fixed per 300
        // config-4 frames); above, the float path is 1-2 % faster at most steps
        // (Δ = 16: 3.95 against 4.03 ms; profiles/r02_config4_packed_lanes.md)
        const int choice = get_option(DCT16A_OPT_UNIFORM_QUANT);   // 0 auto, 1 float, 2 fixed point
        const bool fx_ok = dfx > err_fx && dfx + err_fx < 1.0 / (32.0 * q.step) && wlo < 4294967296.0;
        p.intq = fx_ok && (choice == 2 || (choice == 0 && q.step <= 8)) ? 1 : 0;
        p.hfix = static_cast<uint32_t>(H);   // (1/2 + δ)·2^32 < 2^32
        p.wlo = p.intq ? static_cast<uint32_t>(wlo) : 0u;
    }
    void (*kern)(const CUtensorMap, const CUtensorMap, unsigned long long*, const WParams) =
        codec_warp_kernel<ELEM, UNIFORM, false>;
    if constexpr (UNIFORM)
        if (p.intq) kern = codec_warp_kernel<ELEM, UNIFORM, true>;
    if (int e = smem_optin(reinterpret_cast<const void*>(kern), Cfg::kSmem)) return e;
    long long grid = static_cast<long long>(num_sms()) * Cfg::kCtasPerSm;
    // runs of up to kWClaim tiles, shorter when there are few tiles per resident warp
    // (a small batch then still spreads over many warps)
    p.claim = static_cast<int>(std::min<long long>(kWClaim, std::max<long long>(1, p.n_tiles / (grid * kWWarps * 4))));
    const long long want = (p.n_tiles + kWWarps * p.claim - 1) / (kWWarps * p.claim);
    if (want < grid) grid = want;
    p.total_warps = static_cast<int>(grid) * kWWarps;
    SchedGuard guard(kSchedCodecWarp, st);
    if (guard.error()) return guard.error();
    p.slot = guard.slot();
    kern<<<static_cast<unsigned>(grid), kWWarps * 32, Cfg::kSmem, st>>>(tin, tout,
                                                                        reinterpret_cast<unsigned long long*>(sse), p);
    return static_cast<int>(cudaGetLastError());
}

}  // namespace

int launch_codec_warp(const void* src, const Geom& g, const dct16a_quant& q, void* recon, uint64_t* sse,
                      cudaStream_t st) {
    const bool uni = q.mode == DCT16A_UNIFORM;
    if (g.elem == 1) return uni ? launch_cw<1, true>(src, g, q, recon, sse, st) : launch_cw<1, false>(src, g, q, recon, sse, st);
    return uni ? launch_cw<2, true>(src, g, q, recon, sse, st) : launch_cw<2, false>(src, g, q, recon, sse, st);
}

int launch_codec_allreduce(const void* src, const Geom& g, const dct16a_quant& q, void* recon,
                           uint64_t* const* peers, int n_peers, long long frame_offset, int multicast,
                           cudaStream_t st) {
    const bool uni = q.mode == DCT16A_UNIFORM;
    if (g.elem == 1)
        return uni ? launch_cw<1, true>(src, g, q, recon, nullptr, st, peers, n_peers, frame_offset, multicast)
                   : launch_cw<1, false>(src, g, q, recon, nullptr, st, peers, n_peers, frame_offset, multicast);
    return uni ? launch_cw<2, true>(src, g, q, recon, nullptr, st, peers, n_peers, frame_offset, multicast)
               : launch_cw<2, false>(src, g, q, recon, nullptr, st, peers, n_peers, frame_offset, multicast);
}

}  // namespace dct16a
