// zonal_band.cu — fused zonal codec, warp-cooperative and band-pruned, for
// 8- and 10-bit images and every r (configs 1, 3; the zonal r-sweep's single
// points; r > 136 runs the unpruned BAND = 15 instance): forward -> keep the first r zig-zag
// coefficients with S folded into the weights ->
// inverse (896-901) -> round half away / clamp (reading A6) -> per-image SSE
// (906-910).
//
// A warp owns one 8-block tile (16 rows x 128 px, tile128.cuh) per iteration;
// lane = (block pair bp = lane >> 3: blocks bp and bp + 4 of the tile,
// r8 = lane & 7).  Only the anti-diagonal band k + l <= BAND that holds the
// first r zig-zag positions is computed (BAND 3/5/7/11/15 is a template
// parameter; the compiler removes every network output outside the band and
// every zero input of the inverse, net16.cuh net_inv_head).
// * Row pass (SWAR): lane (bp, r8) runs row t = r8 and t = r8 + 8 of blocks bp
//   and bp + 4 as the two 16-bit lanes of one 32-bit word per pixel (lo + hi·2^16
//   is linear under ±, mod 2^32; |row sum| <= 16·1023 fits a lane for 10-bit
//   too), outputs l <= BAND; the raw SWAR words go to a per-warp smem tile (the
//   transposition buffer of PAPER.md:1082-1090).
// * Column pass, on column l = r8 (and l = r8 + 8 when BAND >= 8) of both
//   blocks, outputs k <= BAND.  8-bit (SWAR): the same words run the column
//   network; only Z is decoded: Z_00 in [0, 65280] zero-extended, every other Z
//   sign-extended from int16 (the K1 ranges).  10-bit (|Z| reaches 261888, too
//   wide for a lane): the row pass biased both lanes by 2^15, the column pass
//   converts each lane to float (one I2F.U16 per value) and runs the network on
//   float pairs (FADD2, exact: |values| < 2^20); the bias leaves 16·2^15 on
//   output 0 only (T·1 = 16·e_0), removed with the DC offset.  W = 2304/(g_k g_l)
//   on the zonal cells, the rounding offset 1152 on the DC input: every pixel of
//   the inverse is N + 1152.
// * Inverse in float32 pairs (FADD2/FFMA2: block bp in .x, block bp + 4 in .y),
//   exact, on N·2^-35: every input W·Z (+1152) and every value the transposed
//   network forms is an integer of magnitude < 1.95e6 (8-bit) / 7.8e6 (10-bit)
//   for any r — the exact maximum of each value, a linear function of the
//   block, over the pixel box (tests/test_exactness_bounds.py) — times 2^-35: a
//   normal float held exactly.  Lane (bp, l) runs the transposed network down
//   column l (inputs k <= BAND, the others compile-time zeros), the smem tile
//   turns columns into rows, lane (bp, r8) runs rows r8, r8 + 8 (inputs
//   l <= BAND).
// * Pixel = floor((N + 1152)/2304) by ONE round-down multiply per two pixels
//   (FMUL2.RM) with c = fl(2^-114/2304): the exact product (N/2304)·2^-149·(1+δ)
//   rounded down to the subnormal grid is floor(N·fl(1/2304))·2^-149, whose bit
//   pattern is that integer (IEEE subnormals, no flush-to-zero).  fl(1/2304) >
//   1/2304 with relative error δ = 7.5e-9, so for 0 <= N < 2^23 the floor is
//   exact; a negative N gives a negative int (sign bit): 8-bit pixels saturate
//   in cvt.pack.sat, 10-bit ones in one relu-min.
// * SSE per row: cvt.pack.sat + vabsdiff4 + dp4a against the original bytes
//   (8-bit) or two integer squares per word (10-bit); the reconstruction
//   overwrites the tile in place and leaves by TMA store.
#include <cuda.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>

#include "internal.h"
#include "net16.cuh"
#include "pack2.cuh"
#include "ptx.cuh"
#include "sched.cuh"
#include "quant.cuh"
#include "tables.cuh"
#include "tile128.cuh"

namespace dct16a {
namespace {

constexpr int kBWarps = 4;
// Per-warp transposition buffers (32-bit words), sharing one region:
//   ty[4 block pairs][16 rows][BAND+1 SWAR words], row pitch kTyRow, pair stride kTyBlock;
//   tu[4 block pairs][16 rows][columns][2 blocks] float, row pitch kTuRow, pair stride kTuBlock.
// The pitches and strides put the lanes of every shared-memory phase on
// distinct banks (one column per lane: 8 columns; two: 16).
template <int ELEM, int BAND>
struct ZCfg {
    static constexpr int kNCol = BAND >= 8 ? 2 : 1;             // columns per lane in the column pass
    static constexpr int kTyRow = kNCol == 1 ? 12 : 20;
    static constexpr int kTyBlock = kNCol == 1 ? 200 : 328;
    static constexpr int kTuRow = kNCol == 1 ? 20 : 36;
    static constexpr int kTuBlock = kNCol == 1 ? 336 : 592;
    static constexpr int kXpose = 4 * (kTuBlock > kTyBlock ? kTuBlock : kTyBlock) * 4;
    // DCT16A_ZB_STAGES1 / DCT16A_ZB_CTAS1: experiment knobs for the 8-bit one-column
    // configuration (tools/dbg/zb_variants.sh, profiles/r02_band_occupancy.md)
#ifdef DCT16A_ZB_STAGES1
    static constexpr int kStages = (ELEM == 1 && kNCol == 1) ? DCT16A_ZB_STAGES1 : 3;
#else
    static constexpr int kStages = (ELEM == 1 && kNCol == 1) ? 4 : 3;   // TMA ring depth per warp
#endif
    static constexpr int kStage = 16 * 128 * ELEM;                       // one tile
    static constexpr int kWarpBytes = kStages * kStage;
    // column weights (kNCol = 2): F2 [16 columns][17] (W·2^-35 for k = 0..15, DC offset)
    static constexpr int kWtab = kNCol == 2 ? 16 * 17 * 8 : 0;
    // CTA smem: [every warp's TMA stages (1024-byte aligned: the swizzle takes
    // address bits 7-9)] [every warp's transposition buffer] [weights]
    // [mbarriers, per-stage tile coordinates]
    static constexpr int kSmem = 1024 + kBWarps * (kWarpBytes + kXpose) + kWtab + kBWarps * kStages * (8 + 16);
    static constexpr int kFit = (227 * 1024) / (kSmem + 1024);
#ifdef DCT16A_ZB_CTAS1
    static constexpr int kCtasMax = (ELEM == 1 && kNCol == 1) ? DCT16A_ZB_CTAS1 : 4;
#else
    static constexpr int kCtasMax = 4;
#endif
    static constexpr int kCtas = kFit < kCtasMax ? kFit : kCtasMax;
};

#ifndef DCT16A_ZB_PROMO
#define DCT16A_ZB_PROMO 0   // input L2 promotion: none (256 B promotion re-reads ~20 % of the input)
#endif
#ifndef DCT16A_ZB_CLAIM
#define DCT16A_ZB_CLAIM 8
#endif
constexpr int kBClaim = DCT16A_ZB_CLAIM;   // consecutive tiles per claim

struct BParams {
    int W, BX, BY, VH, tiles_per_strip;
    long long n_tiles;
    int r;
    int has_recon;
    int slot, total_warps, claim;   // tile scheduler (sched.cuh; slot -1 = static), tiles per claim
};

// Dynamic tile scheduler (sched.cuh, as the forward kernel's): warps claim runs
// of kBClaim consecutive tiles in increasing order from a global counter, so the
// tiles in flight form one compact address window.
__device__ unsigned long long g_zb_sched[kSchedSlots][2];

}  // namespace

template <int ELEM, int BAND>
__global__ void __launch_bounds__(kBWarps * 32, ZCfg<ELEM, BAND>::kCtas)
    zband_kernel(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout,
                 unsigned long long* __restrict__ sse, const BParams p) {
    static_assert(BAND % 2 == 1 && BAND <= 15, "BAND must be odd, <= 15");
    using Cfg = ZCfg<ELEM, BAND>;
    constexpr int kStages = Cfg::kStages;
    constexpr int kNCol = Cfg::kNCol;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = walign1024(smem_raw);
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    uint8_t* wbase = smem + warp * Cfg::kWarpBytes;
    uint32_t* xp = reinterpret_cast<uint32_t*>(smem + kBWarps * Cfg::kWarpBytes + warp * Cfg::kXpose);
    F2* wtab = reinterpret_cast<F2*>(smem + kBWarps * (Cfg::kWarpBytes + Cfg::kXpose));
    uint64_t* bars =
        reinterpret_cast<uint64_t*>(smem + kBWarps * (Cfg::kWarpBytes + Cfg::kXpose) + Cfg::kWtab) + warp * kStages;
    int4* coords = reinterpret_cast<int4*>(smem + kBWarps * (Cfg::kWarpBytes + Cfg::kXpose) + Cfg::kWtab +
                                           kBWarps * kStages * 8) +
                   warp * kStages;
    const uint64_t pol = policy_evict_first();
    unsigned long long* sched = p.slot >= 0 ? g_zb_sched[p.slot] : nullptr;
    Claims claims(sched, static_cast<long long>(blockIdx.x) * kBWarps + warp, static_cast<long long>(gridDim.x) * kBWarps);   // lane 0

    // lane 0: the claim in progress (tiles [next, end)) and its cursor
    long long next = 0, end = 0;
    TileCursor ic;
    // claim the next tile and issue its load into stage `st` (lane 0 only)
    auto issue_next = [&](int st) {
        if (next == end) {
            const long long first = claims.next() * p.claim;
            next = first;
            end = first < p.n_tiles ? min(first + p.claim, p.n_tiles) : first;
            if (first < p.n_tiles) ic.init(p, first);
        }
        if (next < end) {
            coords[st] = make_int4(ic.n, ic.by, ic.tb, 1);
            w_issue_at<ELEM>(&tin, p, ic, wbase + st * Cfg::kStage, &bars[st], pol);
            ++next;
            ic.advance(p);
        } else {
            coords[st] = make_int4(0, 0, 0, 0);
        }
    };
    if (lane == 0) {
        for (int st = 0; st < kStages; ++st) mbar_init(&bars[st], 1);
        fence_mbar_init();
        prefetch_tmap(&tin);
        if (p.has_recon) prefetch_tmap(&tout);
        for (int st = 0; st < kStages - 1; ++st) issue_next(st);
    }

    // The column weights W·2^-35 of the zonal cells (0 elsewhere; the whole
    // inverse runs on N·2^-35, header) for column l, both SWAR lanes: the 8-bit
    // high lane arrives as Z·2^16, so its weight carries 2^-16 (an exact
    // scaling); the 10-bit lanes are decoded separately.  Entry 16: the DC
    // input's offset, 1152·2^-35 for l = 0 (the rounding offset).
    auto col_weight = [&](int k, int l) {
        const float w = zigzag_rank(k, l) < p.r ? static_cast<float>(w_of(k, l)) * 0x1p-35f : 0.0f;
        return F2{make_float2(w, ELEM == 1 ? w * 0x1p-16f : w)};
    };
    auto dc_offset = [&](int l) {
        const float off = l == 0 ? 1152.0f * 0x1p-35f : 0.0f;
        return F2{make_float2(off, off)};
    };
    if constexpr (kNCol == 2) {
        for (int e = threadIdx.x; e < 16 * 17; e += blockDim.x) {
            const int l = e / 17, k = e % 17;
            wtab[e] = k < 16 ? col_weight(k, l) : dc_offset(l);
        }
        __syncthreads();
    } else {
        __syncwarp();
    }

    // lane = (block pair bp = lane >> 3: blocks bp and bp + 4 of the tile, r8 = lane & 7)
    const int bp = lane >> 3;
    const int r8 = lane & 7;   // rows r8, r8 + 8 (row and pixel passes) / column r8 (+ 8) (column pass)
    F2 wl[kNCol == 1 ? BAND + 1 : 1];   // one column per lane: its weights in registers
    F2 dc_off0{make_float2(0.0f, 0.0f)};
    if constexpr (kNCol == 1) {
#pragma unroll
        for (int k = 0; k <= BAND; ++k) wl[k] = col_weight(k, r8);
        dc_off0 = dc_offset(r8);
    }
    // fl(2^-114/2304) = 2^-114·fl(1/2304): N·2^-35 times it is (N/2304)·2^-149 (up to fl)
    const F2 pix_scale{make_float2(0x1p-114f / 2304.0f, 0x1p-114f / 2304.0f)};

    uint32_t* ty = xp + bp * Cfg::kTyBlock;
    float* tu = reinterpret_cast<float*>(xp) + bp * Cfg::kTuBlock;

    unsigned long long acc = 0;
    int cur_n = -1;
    for (int it = 0;; ++it) {
        const int s = it % kStages;
        uint8_t* stage = wbase + s * Cfg::kStage;
        const int4 cd = coords[s];
        if (!cd.w) break;   // claims only grow: every later stage is empty too
        mbar_wait(&bars[s], (it / kStages) & 1);
        TileCursor cc;
        cc.n = cd.x;
        cc.by = cd.y;
        cc.tb = cd.z;
        const int n = cc.n, by = cc.by, x0 = cc.x0();
        if (n != cur_n) {   // image changed (warp-uniform): flush the previous image's SSE
#pragma unroll
            for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (lane == 0 && acc) atomicAdd(sse + cur_n, acc);
            acc = 0;
            cur_n = n;
        }
        const bool valid0 = x0 / 16 + bp < p.BX;
        const bool valid1 = x0 / 16 + bp + 4 < p.BX;

        // ---- row pass: row t of blocks bp and bp + 4 as one SWAR vector, outputs l <= BAND
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int t = r8 + 8 * h;
            uint32_t x[16], y[16];
            if constexpr (ELEM == 1) {
                const uint4 A = *reinterpret_cast<const uint4*>(stage + swz(t, bp));
                const uint4 B = *reinterpret_cast<const uint4*>(stage + swz(t, bp + 4));
                const uint32_t a[4] = {A.x, A.y, A.z, A.w};
                const uint32_t bw[4] = {B.x, B.y, B.z, B.w};
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const uint32_t u = __byte_perm(a[c], bw[c], 0x6420);   // (A0, A2, B0, B2)
                    const uint32_t v = __byte_perm(a[c], bw[c], 0x7531);   // (A1, A3, B1, B3)
                    x[4 * c] = __byte_perm(u, 0u, 0x4240);
                    x[4 * c + 1] = __byte_perm(v, 0u, 0x4240);
                    x[4 * c + 2] = __byte_perm(u, 0u, 0x4341);
                    x[4 * c + 3] = __byte_perm(v, 0u, 0x4341);
                }
            } else {
                int a0, a1, b0, b1;
                row_addr<2>(bp, t, &a0, &a1);
                row_addr<2>(bp + 4, t, &b0, &b1);
                uint32_t wa[8], wb[8];
                load_px<2>(stage, a0, a1, wa);
                load_px<2>(stage, b0, b1, wb);
#pragma unroll
                for (int m = 0; m < 8; ++m) {
                    x[2 * m] = __byte_perm(wa[m], wb[m], 0x5410);       // (A_2m, B_2m)
                    x[2 * m + 1] = __byte_perm(wa[m], wb[m], 0x7632);   // (A_2m+1, B_2m+1)
                }
            }
            net_fwd(x, y);
            if constexpr (ELEM == 2) {
                // both lanes biased by 2^15: two non-negative 16-bit fields (|Y| <= 16368)
#pragma unroll
                for (int q = 0; q <= BAND; ++q) y[q] += 0x80008000u;
            }
            // the SWAR words go to the column pass as they are (lo + hi·2^16 mod 2^32)
            uint32_t* row = ty + t * Cfg::kTyRow;
#pragma unroll
            for (int q = 0; q + 3 <= BAND; q += 4) *reinterpret_cast<uint4*>(row + q) = make_uint4(y[q], y[q + 1], y[q + 2], y[q + 3]);
            if constexpr ((BAND + 1) % 4 == 2)
                *reinterpret_cast<uint2*>(row + BAND - 1) = make_uint2(y[BAND - 1], y[BAND]);
        }
        __syncwarp();

        // ---- column pass on column l of both blocks, outputs k <= BAND; weights; inverse down the column
        {
            uint32_t cwv[kNCol][16];
#pragma unroll
            for (int c2 = 0; c2 < kNCol; ++c2)
#pragma unroll
                for (int t = 0; t < 16; ++t) cwv[c2][t] = ty[t * Cfg::kTyRow + r8 + 8 * c2];
            __syncwarp();   // every lane has read ty before tu (same buffer) is written
#pragma unroll
            for (int c2 = 0; c2 < kNCol; ++c2) {
                const int l = r8 + 8 * c2;
                if (c2 == 1 && l > BAND) continue;   // no zonal cell in this column
                F2 c[16];
                if constexpr (ELEM == 1) {
                    uint32_t z[16];
                    net_fwd(cwv[c2], z);
                    const bool dc_lane = l == 0;   // Z_00 in [0, 65280]: unsigned
#pragma unroll
                    for (int k = 0; k <= BAND; ++k) {
                        // z[k] = Z_lo + Z_hi·2^16 (mod 2^32); Z_00 in [0, 65280], every other Z in int16
                        const bool uns = k == 0 && dc_lane;
                        const int lo = uns ? static_cast<int>(z[k] & 0xFFFFu) : static_cast<int>(static_cast<int16_t>(z[k] & 0xFFFFu));
                        const uint32_t hs = z[k] - static_cast<uint32_t>(lo);   // Z_hi·2^16
                        const float hf = uns ? static_cast<float>(hs) : static_cast<float>(static_cast<int>(hs));
                        const F2 w = kNCol == 1 ? wl[k < BAND + 1 ? k : 0] : wtab[l * 17 + k];
                        const F2 off = k == 0 ? (kNCol == 1 ? dc_off0 : wtab[l * 17 + 16]) : F2{make_float2(0.0f, 0.0f)};
                        // exact in float: W·Z + 1152 and every later value are integers below 2^21 (header)
                        c[k] = fma2(F2{make_float2(static_cast<float>(lo), hf)}, w, off);
                    }
                } else {
                    F2 cf[16], zf[16];
#pragma unroll
                    for (int t = 0; t < 16; ++t)
                        cf[t] = F2{make_float2(static_cast<float>(cwv[c2][t] & 0xFFFFu), static_cast<float>(cwv[c2][t] >> 16))};
                    net_fwd(cf, zf);
                    zf[0] = zf[0] - F2{make_float2(524288.0f, 524288.0f)};   // 16·2^15 of the bias (exact: < 2^20)
#pragma unroll
                    for (int k = 0; k <= BAND; ++k) {
                        const F2 w = kNCol == 1 ? wl[k < BAND + 1 ? k : 0] : wtab[l * 17 + k];
                        const F2 off = k == 0 ? (kNCol == 1 ? dc_off0 : wtab[l * 17 + 16]) : F2{make_float2(0.0f, 0.0f)};
                        c[k] = fma2(zf[k], w, off);
                    }
                }
                F2 u[16];
                net_inv_head<BAND + 1>(c, u);
#pragma unroll
                for (int i = 0; i < 16; ++i) *reinterpret_cast<float2*>(tu + i * Cfg::kTuRow + 2 * l) = u[i].v;
            }
        }
        __syncwarp();

        // ---- inverse along row i of both blocks, pixels, SSE, in-place reconstruction
        // (the tile's SSE in 32 bits: at most 4 rows x 16 x maxpix^2 per lane)
        uint32_t etile = 0;
        const uint32_t m0 = valid0 ? 0xFFFFFFFFu : 0u, m1 = valid1 ? 0xFFFFFFFFu : 0u;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int i = r8 + 8 * h;
            F2 v[16], a[16];
#pragma unroll
            for (int j = 0; j <= BAND; j += 2) {
                const float4 q4 = *reinterpret_cast<const float4*>(tu + i * Cfg::kTuRow + 2 * j);
                v[j] = F2{make_float2(q4.x, q4.y)};
                v[j + 1] = F2{make_float2(q4.z, q4.w)};
            }
            net_inv_head<BAND + 1>(v, a);
            int pa[16], pb[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                // floor((N + 1152)/2304) for both blocks by one round-down multiply into
                // the subnormal range: the bits of the result are the integer itself
                const float2 r = fmul2_rd_keep_subnormal(a[j].v, pix_scale.v);
                pa[j] = __float_as_int(r.x);
                pb[j] = __float_as_int(r.y);
            }
            const bool row_ok = by * 16 + i < p.VH;
#pragma unroll
            for (int blk = 0; blk < 2; ++blk) {
                const int* pv = blk ? pb : pa;
                uint32_t e = 0;
                if constexpr (ELEM == 1) {
                    uint32_t o[4];
#pragma unroll
                    for (int c4 = 0; c4 < 4; ++c4)
                        o[c4] = pack2_sat_u8(pv[4 * c4 + 1], pv[4 * c4], pack2_sat_u8(pv[4 * c4 + 3], pv[4 * c4 + 2], 0u));
                    uint4* cell = reinterpret_cast<uint4*>(stage + swz(i, bp + 4 * blk));
                    const uint4 orig = *cell;
                    const uint32_t ow[4] = {orig.x, orig.y, orig.z, orig.w};
#pragma unroll
                    for (int c4 = 0; c4 < 4; ++c4) {
                        const uint32_t dd = __vabsdiffu4(o[c4], ow[c4]);
                        e = __dp4a(dd, dd, e);
                    }
                    if (p.has_recon) *cell = make_uint4(o[0], o[1], o[2], o[3]);
                } else {
                    int c0, c1;
                    row_addr<2>(bp + 4 * blk, i, &c0, &c1);
                    uint32_t ow[8], o[8];
                    load_px<2>(stage, c0, c1, ow);
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        // clamp to [0, 1023] (a negative N left a negative int)
                        const int p0 = __vimin_s32_relu(pv[2 * q], 1023), p1 = __vimin_s32_relu(pv[2 * q + 1], 1023);
                        o[q] = __byte_perm(p0, p1, 0x5410);
                        const int d0 = p0 - static_cast<int>(ow[q] & 0xFFFFu);
                        const int d1 = p1 - static_cast<int>(ow[q] >> 16);
                        e += static_cast<uint32_t>(d0 * d0 + d1 * d1);
                    }
                    if (p.has_recon) {
                        *reinterpret_cast<uint4*>(stage + c0) = make_uint4(o[0], o[1], o[2], o[3]);
                        *reinterpret_cast<uint4*>(stage + c1) = make_uint4(o[4], o[5], o[6], o[7]);
                    }
                }
                etile += e & (blk ? m1 : m0) & (row_ok ? 0xFFFFFFFFu : 0u);
            }
        }
        acc += etile;
        __syncwarp();
        if (lane == 0) {
            if (p.has_recon) {
                fence_async_smem();
                w_store_at<ELEM>(&tout, p, cc, stage);
                bulk_commit();
                bulk_wait_read<1>();   // the store of tile tix-1 has left the stage refilled next
            }
            issue_next((it + kStages - 1) % kStages);
        }
        __syncwarp();
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
        if (acc) atomicAdd(sse + cur_n, acc);
        if (p.has_recon) bulk_wait<0>();
        claims_done(sched, p.total_warps);   // every warp has claimed past the end
    }
}

namespace {

template <int ELEM, int BAND>
int launch_zb(const void* src, const Geom& g, int r, void* recon, uint64_t* sse, cudaStream_t st) {
    using Cfg = ZCfg<ELEM, BAND>;
    CUtensorMap tin, tout;
    const uint64_t dims[3] = {uint64_t(g.W), uint64_t(g.H), uint64_t(g.N)};
    const uint64_t strides[2] = {uint64_t(g.pitch), uint64_t(g.istride)};
    const uint32_t box[3] = {uint32_t(128 / ELEM), 16u, 1u};
    const CUtensorMapDataType dt = ELEM == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_UINT16;
    // 8-bit: no L2 promotion (256 B promotion re-reads ~20 % of the input); 10-bit
    // tiles are two adjacent 128-byte boxes, where 256 B promotion costs nothing
    if (encode_tiled(&tin, dt, 3, src, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B,
                     ELEM == 1 ? static_cast<CUtensorMapL2promotion>(DCT16A_ZB_PROMO) : CU_TENSOR_MAP_L2_PROMOTION_L2_256B))
        return DCT16A_ECUDA;
    if (recon) {
        if (encode_tiled(&tout, dt, 3, recon, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_NONE))
            return DCT16A_ECUDA;
    } else {
        tout = tin;
    }
    BParams p{};
    p.W = g.W;
    p.BX = g.BX;
    p.BY = g.BY;
    p.VH = g.VH;
    p.tiles_per_strip = (g.BX + kWTile - 1) / kWTile;
    p.n_tiles = static_cast<long long>(g.N) * g.BY * p.tiles_per_strip;
    p.r = r;
    p.has_recon = recon != nullptr;
    if (int e = smem_optin(reinterpret_cast<const void*>(zband_kernel<ELEM, BAND>), Cfg::kSmem)) return e;
    long long grid = static_cast<long long>(num_sms()) * Cfg::kCtas;
    // runs of up to kBClaim tiles, shorter when there are few tiles per resident warp
    // (a small batch then still spreads over many warps)
    p.claim = static_cast<int>(std::min<long long>(kBClaim, std::max<long long>(1, p.n_tiles / (grid * kBWarps * 4))));
    const long long want = (p.n_tiles + kBWarps * p.claim - 1) / (kBWarps * p.claim);
    if (want < grid) grid = want;
    p.total_warps = static_cast<int>(grid) * kBWarps;
    SchedGuard guard(kSchedBand, st);
    if (guard.error()) return guard.error();
    p.slot = guard.slot();
    zband_kernel<ELEM, BAND><<<static_cast<unsigned>(grid), kBWarps * 32, Cfg::kSmem, st>>>(
        tin, tout, reinterpret_cast<unsigned long long*>(sse), p);
    return static_cast<int>(cudaGetLastError());
}

template <int ELEM>
int launch_zb_e(const void* src, const Geom& g, int r, void* recon, uint64_t* sse, cudaStream_t st) {
    const int band = zonal_band(r);
    if (band <= 3) return launch_zb<ELEM, 3>(src, g, r, recon, sse, st);
    if (band <= 5) return launch_zb<ELEM, 5>(src, g, r, recon, sse, st);
    if (band <= 7) return launch_zb<ELEM, 7>(src, g, r, recon, sse, st);
    if (band <= 11) return launch_zb<ELEM, 11>(src, g, r, recon, sse, st);
    return launch_zb<ELEM, 15>(src, g, r, recon, sse, st);   // also every r > 136 (band > 15)
}

}  // namespace

// Smallest anti-diagonal band holding the first r zig-zag positions.
int zonal_band(int r) {
    int d = 0;
    while ((d + 1) * (d + 2) / 2 < r) ++d;   // cells with k + l <= d: (d+1)(d+2)/2 (d <= 15)
    return d;
}

// The band kernel covers every r, 8- and 10-bit: r <= 136 on the smallest band
// k + l <= BAND holding the zig-zag prefix; beyond (k + l reaching 16..30) on
// BAND = 15, which computes every output of both networks (nothing left to
// prune) and keeps the first r cells through the weights (zero elsewhere).
bool zonal_band_applies(const Geom& g, int r) { (void)g; return r >= 1 && r <= 256; }

// Callers check zonal_band_applies first.
int launch_zonal_band(const void* src, const Geom& g, int r, void* recon, uint64_t* sse, cudaStream_t st) {
    if (r < 1 || r > 256) return DCT16A_EDOMAIN;
    return g.elem == 1 ? launch_zb_e<1>(src, g, r, recon, sse, st) : launch_zb_e<2>(src, g, r, recon, sse, st);
}

}  // namespace dct16a
