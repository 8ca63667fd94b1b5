// zonal_band.cu — fused zonal codec for 8-bit images with r <= 36 (configs 1,
// 3), warp-cooperative and band-pruned: forward -> keep the
// first r zig-zag coefficients with S folded into the weights (PAPER.md:333-344,
// 882-894) -> inverse (896-901) -> round half away / clamp (reading A6) ->
// per-image SSE (906-910).
//
// A warp owns one 8-block tile (16 rows x 128 px, tile128.cuh) per iteration;
// lane = (block b = lane & 7, quarter q = lane >> 3).  Only the anti-diagonal
// band k + l <= BAND that holds the first r zig-zag positions is computed
// (BAND 3/5/7 is a template parameter; the compiler removes every network
// output outside the band and every zero input of the inverse).
// * Row pass (SWAR): lane (b, q) runs rows (q, q+8) and (q+4, q+12) of block b
//   as two 16-bit lanes of one 32-bit word (lo + hi·2^16 is linear under ±),
//   so 128 rows take 2 networks per lane; outputs l <= BAND, biased by 2^15 so
//   the halves are non-negative and are repacked by PRMT into column-pair words
//   (Y[t][2p], Y[t][2p+1]) — the transposition buffer of PAPER.md:1082-1090 is
//   a per-warp smem tile.
// * Column pass (SWAR): lane (b, p = q) runs column pair (2p, 2p+1) down the 16
//   rows, outputs k <= BAND; Z_00 in [0, 65280] is decoded unsigned, every other
//   Z in int16 (the K1 ranges).  W = 2304/(g_k g_l) on the zonal cells, the
//   rounding offset 1152 on the DC input: every pixel of the inverse is N + 1152.
// * Inverse in int32 (exact: |N| < 2^23 for 8-bit input): lane (b, p) runs the
//   transposed network down its two columns (inputs k <= BAND), the smem tile
//   turns columns into rows, lane (b, q) runs rows q, q+4, q+8, q+12 (inputs
//   l <= BAND).  pixel = floor((N + 1152)/2304) by one I2F and one round-down
//   FMA onto 2^23 (exact: fl(1/2304) > 1/2304 with relative error 7.5e-9, so
//   for 0 <= x < 2^23 the product never falls below an integer it should reach
//   nor reaches one it should not; negative results saturate to 0 in the pack).
// * SSE per row: cvt.pack.sat + vabsdiff4 + dp4a against the original bytes;
//   the reconstruction overwrites the tile in place and leaves by TMA store.
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

#ifndef DCT16A_ZB_STAGES
#define DCT16A_ZB_STAGES 3
#endif
#ifndef DCT16A_ZB_CTAS
#define DCT16A_ZB_CTAS 4
#endif
constexpr int kBWarps = 4;
constexpr int kBStages = DCT16A_ZB_STAGES;
constexpr int kBStage = 16 * 128;   // one u8 tile
// per-warp transposition words: ty[8 blocks][16 rows][4 column-pair words]
// (block stride 68) and tu[8 blocks][16 rows][8 int32] (block stride 132) share
// one buffer; the strides put the 8 blocks of a quarter-warp on distinct banks
constexpr int kTyBlock = 68;
constexpr int kTuBlock = 132;
constexpr int kBXpose = 5120;   // >= 8·132·4 = 4224 B, keeps every stage 1024-byte aligned
constexpr int kBWarpBytes = kBStages * kBStage + kBXpose;
static_assert(kBWarpBytes % 1024 == 0, "stages must stay 1024-byte aligned");
static_assert(8 * kTuBlock * 4 <= kBXpose, "transposition buffer too small");
constexpr int kBSmem = 1024 + kBWarps * kBWarpBytes + kBWarps * kBStages * 8;

struct BParams {
    int W, BX, BY, VH, tiles_per_strip;
    long long n_tiles, chunk;   // tiles, tiles per warp
    int r;
    int has_recon;
};

}  // namespace

template <int BAND>
__global__ void __launch_bounds__(kBWarps * 32, DCT16A_ZB_CTAS)
    zband_kernel(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout,
                 unsigned long long* __restrict__ sse, const BParams p) {
    constexpr int NP = BAND / 2 + 1;   // column pairs covering l <= BAND (BAND odd)
    static_assert(BAND % 2 == 1 && BAND <= 7, "BAND must be 3, 5 or 7");
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = walign1024(smem_raw);
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    uint8_t* wbase = smem + warp * kBWarpBytes;
    uint32_t* xp = reinterpret_cast<uint32_t*>(wbase + kBStages * kBStage);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kBWarps * kBWarpBytes) + warp * kBStages;

    const long long gw = static_cast<long long>(blockIdx.x) * kBWarps + warp;
    const long long t0 = gw * p.chunk;
    long long t1 = t0 + p.chunk;
    if (t1 > p.n_tiles) t1 = p.n_tiles;
    const uint64_t pol = policy_evict_first();

    if (lane == 0) {
        for (int s = 0; s < kBStages; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
        prefetch_tmap(&tin);
        if (p.has_recon) prefetch_tmap(&tout);
        TileCursor ic;
        ic.init(p, t0);
        for (int s = 0; s < kBStages - 1; ++s) {
            if (t0 + s < t1) w_issue_at<1>(&tin, p, ic, wbase + s * kBStage, &bars[s], pol);
            ic.advance(p);
        }
    }
    __syncwarp();

    const int b = lane & 7;    // block of the tile
    const int q = lane >> 3;   // row quarter (row and pixel passes) / column pair (column pass)
    // column pass constants: weights of columns 2q, 2q+1 (0 outside the zonal set)
    int w0[BAND + 1], w1s[BAND + 1];
#pragma unroll
    for (int k = 0; k <= BAND; ++k) {
        w0[k] = zigzag_rank(k, 2 * q) < p.r ? w_of(k, 2 * q) : 0;
        w1s[k] = zigzag_rank(k, 2 * q + 1) < p.r ? (w_of(k, 2 * q + 1) << 16) : 0;   // ·2^16 for mulhi
    }
    const bool dc_unsigned = q == 0;                       // Z_00 in [0, 65280] is decoded unsigned
    const int dc_off = q == 0 ? 1152 : 0;                  // rounding offset on the DC input
    const float inv2304 = 1.0f / 2304.0f;

    uint32_t* ty = xp + b * kTyBlock;
    uint32_t* tu = xp + b * kTuBlock;

    unsigned long long acc = 0;
    int cur_n = -1;
    int it = 0;
    TileCursor cc, nc;   // the tile being consumed and the one kBStages - 1 ahead
    cc.init(p, t0);
    nc.init(p, t0 + kBStages - 1);
    for (long long tix = t0; tix < t1; ++tix, ++it, cc.advance(p), nc.advance(p)) {
        const int s = it % kBStages;
        uint8_t* stage = wbase + s * kBStage;
        mbar_wait(&bars[s], (it / kBStages) & 1);
        const int n = cc.n, by = cc.by, x0 = cc.x0();
        if (n != cur_n) {   // image changed (warp-uniform): flush the previous image's SSE
#pragma unroll
            for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (lane == 0 && acc) atomicAdd(sse + cur_n, acc);
            acc = 0;
            cur_n = n;
        }
        const bool bvalid = x0 / 16 + b < p.BX;

        // ---- row pass: rows (q + 4pr, q + 4pr + 8) as one SWAR vector, outputs l <= BAND
#pragma unroll
        for (int pr = 0; pr < 2; ++pr) {
            const int t = q + 4 * pr;
            const uint4 A = *reinterpret_cast<const uint4*>(stage + swz(t, b));
            const uint4 B = *reinterpret_cast<const uint4*>(stage + swz(t + 8, b));
            const uint32_t a[4] = {A.x, A.y, A.z, A.w};
            const uint32_t bw[4] = {B.x, B.y, B.z, B.w};
            uint32_t x[16], y[16];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const uint32_t u = __byte_perm(a[c], bw[c], 0x6420);   // (A0, A2, B0, B2)
                const uint32_t v = __byte_perm(a[c], bw[c], 0x7531);   // (A1, A3, B1, B3)
                x[4 * c] = __byte_perm(u, 0u, 0x4240);
                x[4 * c + 1] = __byte_perm(v, 0u, 0x4240);
                x[4 * c + 2] = __byte_perm(u, 0u, 0x4341);
                x[4 * c + 3] = __byte_perm(v, 0u, 0x4341);
            }
            net_fwd(x, y);
            uint32_t ra[NP], rb[NP];
#pragma unroll
            for (int pp = 0; pp < NP; ++pp) {
                // |Y| <= 4080: +2^15 per lane keeps both halves non-negative, so each
                // half is the exact biased value and PRMT can regroup them
                const uint32_t y0 = y[2 * pp] + 0x80008000u, y1 = y[2 * pp + 1] + 0x80008000u;
                ra[pp] = __byte_perm(y0, y1, 0x5410);   // row t:     (Y[t][2pp], Y[t][2pp+1])
                rb[pp] = __byte_perm(y0, y1, 0x7632);   // row t + 8
            }
            if constexpr (NP == 4) {
                *reinterpret_cast<uint4*>(ty + t * 4) = make_uint4(ra[0], ra[1], ra[2], ra[3]);
                *reinterpret_cast<uint4*>(ty + (t + 8) * 4) = make_uint4(rb[0], rb[1], rb[2], rb[3]);
            } else {
#pragma unroll
                for (int pp = 0; pp < NP; ++pp) {
                    ty[t * 4 + pp] = ra[pp];
                    ty[(t + 8) * 4 + pp] = rb[pp];
                }
            }
        }
        __syncwarp();

        // ---- column pass on column pair (2q, 2q+1), outputs k <= BAND; weights; inverse down the columns
        {
            uint32_t cw[16], z[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) cw[k] = ty[k * 4 + q];
            __syncwarp();   // every lane has read ty before tu (same buffer) is written
            net_fwd(cw, z);
            int c0[16], c1[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                c0[k] = 0;
                c1[k] = 0;
            }
#pragma unroll
            for (int k = 0; k <= BAND; ++k) {
                // the 2^15 input bias adds 2^15·(sum of row k of T) per lane: 2^19 for k = 0, 0 otherwise
                const uint32_t wd = k == 0 ? z[0] - 0x00080000u : z[k];
                const int lo = k == 0 && dc_unsigned ? static_cast<int>(wd & 0xFFFFu)
                                                     : static_cast<int>(static_cast<int16_t>(wd & 0xFFFFu));
                const int hs = static_cast<int>(wd - static_cast<uint32_t>(lo));   // Z_hi·2^16
                c0[k] = lo * w0[k] + (k == 0 ? dc_off : 0);
                c1[k] = __mulhi(hs, w1s[k]);                                      // Z_hi·W
            }
            int u0[16], u1[16];
            net_inv(c0, u0);
            net_inv(c1, u1);
#pragma unroll
            for (int i = 0; i < 16; ++i)
                *reinterpret_cast<int2*>(tu + i * 8 + 2 * q) = make_int2(u0[i], u1[i]);
        }
        __syncwarp();

        // ---- inverse along the rows q, q+4, q+8, q+12, pixels, SSE, in-place reconstruction
#pragma unroll
        for (int s4 = 0; s4 < 4; ++s4) {
            const int i = q + 4 * s4;
            int v[16], a[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = 0;
            {
                const int4 v0 = *reinterpret_cast<const int4*>(tu + i * 8);
                v[0] = v0.x; v[1] = v0.y; v[2] = v0.z; v[3] = v0.w;
                if (BAND >= 4) {
                    const int4 v1 = *reinterpret_cast<const int4*>(tu + i * 8 + 4);
                    v[4] = v1.x; v[5] = v1.y;
                    if (BAND >= 6) { v[6] = v1.z; v[7] = v1.w; }
                }
            }
            net_inv(v, a);
            int pv[16];
#pragma unroll
            for (int j = 0; j < 16; ++j)
                pv[j] = static_cast<int>(__float_as_uint(__fmaf_rd(static_cast<float>(a[j]), inv2304, 8388608.0f)) -
                                         0x4B000000u);
            uint32_t o[4];
#pragma unroll
            for (int c = 0; c < 4; ++c)
                o[c] = pack2_sat_u8(pv[4 * c + 1], pv[4 * c], pack2_sat_u8(pv[4 * c + 3], pv[4 * c + 2], 0u));
            uint4* cell = reinterpret_cast<uint4*>(stage + swz(i, b));
            const uint4 orig = *cell;
            uint32_t e = 0;
            const uint32_t ow[4] = {orig.x, orig.y, orig.z, orig.w};
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const uint32_t dd = __vabsdiffu4(o[c], ow[c]);
                e = __dp4a(dd, dd, e);
            }
            if (bvalid && by * 16 + i < p.VH) acc += e;
            if (p.has_recon) *cell = make_uint4(o[0], o[1], o[2], o[3]);
        }
        __syncwarp();
        if (lane == 0) {
            if (p.has_recon) {
                fence_async_smem();
                w_store_at<1>(&tout, p, cc, stage);
                bulk_commit();
                bulk_wait_read<1>();   // the store of tile tix-1 has left the stage refilled next
            }
            const long long nt = tix + kBStages - 1;
            if (nt < t1) w_issue_at<1>(&tin, p, nc, wbase + ((it + kBStages - 1) % kBStages) * kBStage,
                                       &bars[(it + kBStages - 1) % kBStages], pol);
        }
        __syncwarp();
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
        if (acc) atomicAdd(sse + cur_n, acc);
        if (p.has_recon) bulk_wait<0>();
    }
}

namespace {

template <int BAND>
int launch_zb(const void* src, const Geom& g, int r, void* recon, uint64_t* sse, cudaStream_t st) {
    CUtensorMap tin, tout;
    const uint64_t dims[3] = {uint64_t(g.W), uint64_t(g.H), uint64_t(g.N)};
    const uint64_t strides[2] = {uint64_t(g.pitch), uint64_t(g.istride)};
    const uint32_t box[3] = {128u, 16u, 1u};
    if (encode_tiled(&tin, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, src, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B))
        return DCT16A_ECUDA;
    if (recon) {
        if (encode_tiled(&tout, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, recon, dims, strides, box,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE))
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
    if (int e = smem_optin(reinterpret_cast<const void*>(zband_kernel<BAND>), kBSmem)) return e;
    long long warps = static_cast<long long>(num_sms()) * DCT16A_ZB_CTAS * kBWarps;
    if (warps > p.n_tiles) warps = p.n_tiles;
    p.chunk = (p.n_tiles + warps - 1) / warps;
    const long long grid = (warps + kBWarps - 1) / kBWarps;
    zband_kernel<BAND><<<static_cast<unsigned>(grid), kBWarps * 32, kBSmem, st>>>(
        tin, tout, reinterpret_cast<unsigned long long*>(sse), p);
    return static_cast<int>(cudaGetLastError());
}

}  // namespace

// Returns 1 if the band kernel does not cover this case (10-bit, or r > 36).
int launch_zonal_band(const void* src, const Geom& g, int r, void* recon, uint64_t* sse, cudaStream_t st) {
    if (g.elem != 1) return 1;
    const int band = zonal_band(r);
    if (band <= 3) return launch_zb<3>(src, g, r, recon, sse, st);
    if (band <= 5) return launch_zb<5>(src, g, r, recon, sse, st);
    if (band <= 7) return launch_zb<7>(src, g, r, recon, sse, st);
    return 1;
}

}  // namespace dct16a
