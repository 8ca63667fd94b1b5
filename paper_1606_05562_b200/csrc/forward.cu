// forward.cu — K1: the standalone forward 2-D transform Z = T·X·Tᵀ over every
// 16x16 block (row pass, transposition, column pass as in
// the paper's 2-D architecture), int32 block-major out.
//
// B200 design:
//  * one thread owns one 16x16 block; a warp owns a tile of 32 horizontally
//    adjacent blocks of one 16-row strip; warps are persistent and claim
//    tiles in increasing order from a global counter (dynamic scheduler
//    below), so the tiles in flight form one compact address window;
//  * TMA (cp.async.bulk.tensor) streams the 16-row strip tile into a 2-stage
//    per-warp smem ring (mbarrier complete_tx); pixels are read back with
//    128-bit ld.shared (conflict-free: a phase of 8 lanes reads 128 contiguous
//    bytes);
//  * both 1-D passes run the 60-add network of Eq. (1) on 16-bit SWAR pairs
//    (two vectors per 32-bit register, lo + hi·2^16), so the 2-D transform
//    costs 8+8 networks = 960 adds per block instead of 1920.  The column pass
//    runs first (pairs of adjacent columns, |T·X| <= 16·maxpix fits a lane);
//    the transposition buffer of the paper is a register byte-permute (PRMT)
//    that turns "column pair of one row" into "row pair of one column";
//    the row pass then yields two rows of Z per network (8-bit: Z_00 in
//    [0, 65280] is the only entry outside int16 and is decoded unsigned);
//  * each Z row pair (128 B per block) is staged in smem in the TMA 128-byte
//    swizzle (conflict-free STS); by default (store mode 5) the whole 32 KB
//    tile leaves in one TMA tensor store (bulk async-group), the other modes
//    below store 4-16 KB pieces from alternating buffers.
#include <cuda.h>
#include <stdint.h>
#include <stdlib.h>

#include <atomic>

#include "internal.h"
#include "net16.cuh"
#include "ptx.cuh"
#include "sched.cuh"

namespace dct16a {
namespace {

constexpr int kTile = 32;    // blocks per warp tile = lanes

// Output paths (SM = store mode):
//  0: TMA tensor store of one Z row pair (32 blocks x 128 B = 4 KB), 2 buffers
//  1: as 0 with 4 buffers
//  2: smem transpose + coalesced 128-bit st.global (LSU path), 1 buffer
//  3: TMA tensor store of two row pairs (8 KB), 2 buffers
//  4: TMA tensor store of four row pairs (16 KB), 2 buffers
//  5: TMA tensor store of the whole tile (8 row pairs, 32 KB), 1 buffer
//  6: as 5 with 2 buffers (2 warps per SM)
//  7: as 5 with a 3-stage input ring
//  8: 16-bit coefficients (dct16a_forward16): the whole tile (32 blocks x
//     512 B = 16 KB) in one TMA tensor store, 64-byte swizzle, 1 buffer
template <int SM>
struct StoreCfg {
    static constexpr bool kOut16 = SM == 8;
    static constexpr int kBufs = SM == 1 ? 4 : ((SM == 2 || SM == 5 || SM == 7 || SM == 8) ? 1 : 2);
    static constexpr int kPairs = SM == 3 ? 2 : (SM == 4 ? 4 : (SM >= 5 ? 8 : 1));   // row pairs per store
    static constexpr int kBytes = kTile * (kOut16 ? 64 : 128) * kPairs;
    static constexpr int kStages = SM == 7 ? 3 : 2;   // input ring depth per warp
};

template <int ELEM, int SM>
struct FwdCfg {
    static constexpr int kStageBytes = 16 * 512 * ELEM;   // 16 rows x 512 px
    static constexpr int kStages = StoreCfg<SM>::kStages;
    static constexpr int kWarpBytes = kStages * kStageBytes + StoreCfg<SM>::kBufs * StoreCfg<SM>::kBytes;
    // as many warps as the 227 KB of shared memory per SM allows, 4 or 5 per CTA
    static constexpr int kWarpsPerSm = (227 * 1024 - 2048) / kWarpBytes;
    static constexpr int kWarps = kWarpsPerSm >= 8 ? 4 : (kWarpsPerSm >= 5 ? 5 : kWarpsPerSm);
    static constexpr int kMinCtas = kWarpsPerSm >= 8 ? 2 : 1;
    static constexpr int kSmem = 1024 + kWarps * kWarpBytes + kWarps * kStages * 8;
};

struct FwdParams {
    int W, BX, BY, tiles_per_strip, box_w;
    long long n_tiles;
    int slot;            // tile-scheduler slot, -1 = static schedule (sched.cuh)
    int total_warps;
};

// Dynamic tile scheduler (sched.cuh): warps claim tiles in increasing order
// from a global counter, so the tiles in flight form one compact address window
// (the static stride schedule lets warps drift apart and spreads the concurrent
// writes over many DRAM pages: 5.6 vs 6.2 TB/s for the same byte mix in
// tools/dbg/mix_dynamic.cu).  A launch captured into a CUDA graph uses the
// static schedule.
__device__ unsigned long long g_fwd_sched[kSchedSlots][2];

// Pad the dynamic smem base to 1024 B (128-byte swizzle atoms) while keeping
// the pointer derived from the __shared__ array, so the compiler emits LDS/STS.
__device__ __forceinline__ uint8_t* align1024(uint8_t* smem_raw) {
    return smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
}

// Issue the TMA loads of tile `tix` into `stage` (one elected lane).
template <int ELEM>
__device__ __forceinline__ void issue_tile(const CUtensorMap* tin, const FwdParams& p, long long tix,
                                           uint8_t* stage, uint64_t* bar, uint64_t pol) {
    const long long strip = tix / p.tiles_per_strip;
    const int tb = static_cast<int>(tix - strip * p.tiles_per_strip);
    const int n = static_cast<int>(strip / p.BY);
    const int by = static_cast<int>(strip - static_cast<long long>(n) * p.BY);
    const int x0 = tb * kTile * 16;
    const int nbox_max = 512 / p.box_w;
    int nbox = 0;
    for (int h = 0; h < nbox_max; ++h)
        if (x0 + h * p.box_w < p.W) ++nbox;
    mbar_arrive_expect_tx(bar, static_cast<uint32_t>(nbox * 16 * p.box_w * ELEM));
    for (int h = 0; h < nbox; ++h)
        tma_load_3d(stage + h * 16 * p.box_w * ELEM, tin, bar, x0 + h * p.box_w, by * 16, n, pol);
}

}  // namespace

template <int ELEM, int SM>
__global__ void __launch_bounds__(FwdCfg<ELEM, SM>::kWarps * 32, FwdCfg<ELEM, SM>::kMinCtas)
    fwd_kernel(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout,
               int32_t* __restrict__ coef, const FwdParams p) {
    using Cfg = FwdCfg<ELEM, SM>;
    using SC = StoreCfg<SM>;
    constexpr int kStages = Cfg::kStages;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = align1024(smem_raw);
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    uint8_t* wbase = smem + warp * Cfg::kWarpBytes;
    uint8_t* outb = wbase + kStages * Cfg::kStageBytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::kWarps * Cfg::kWarpBytes) + warp * kStages;

    const long long gw = static_cast<long long>(blockIdx.x) * Cfg::kWarps + warp;
    const long long nw = static_cast<long long>(gridDim.x) * Cfg::kWarps;
    const uint64_t pol = policy_evict_first();
    unsigned long long* sched = p.slot >= 0 ? g_fwd_sched[p.slot] : nullptr;
    Claims claims(sched, gw, nw);   // lane 0 only

    // tile of pipeline stage s (lane 0 holds the truth; broadcast when used)
    long long ring[kStages];
    if (lane == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
        prefetch_tmap(&tin);
        prefetch_tmap(&tout);
        for (int s = 0; s < kStages; ++s) {
            const long long t = claims.next();
            ring[s] = t;
            if (t < p.n_tiles) issue_tile<ELEM>(&tin, p, t, wbase + s * Cfg::kStageBytes, &bars[s], pol);
        }
    }
    __syncwarp();

    // this lane's block inside the tile: box h, column offset inside the box
    const int px = lane * 16;
    const int lane_off = (px / p.box_w) * 16 * p.box_w * ELEM + (px % p.box_w) * ELEM;
    const int row_pitch = p.box_w * ELEM;
    const int box_b = p.BX < kTile ? p.BX : kTile;   // blocks per output box (dim 1)
    int obuf = 0;
    int it = 0;
    for (;; ++it) {
        const int s = it % kStages;
        long long tix = 0;
#pragma unroll
        for (int q = 0; q < kStages; ++q) tix = q == s ? ring[q] : tix;
        tix = __shfl_sync(0xffffffffu, tix, 0);
        if (tix >= p.n_tiles) break;
        uint8_t* stage = wbase + s * Cfg::kStageBytes;
        mbar_wait(&bars[s], (it / kStages) & 1);

        const long long strip = tix / p.tiles_per_strip;
        const int bx0 = static_cast<int>(tix - strip * p.tiles_per_strip) * kTile;
        const int nvalid = p.BX - bx0 < kTile ? p.BX - bx0 : kTile;   // blocks of this tile inside the strip
        int4* tile_dst = reinterpret_cast<int4*>(coef) + (strip * p.BX + bx0) * 64 + (lane & 7) + (lane >> 3) * 64;

        // ---- column pass (SWAR: column pairs (2m, 2m+1) of one row per register)
        uint32_t o[8][16];
        if constexpr (ELEM == 1) {
            uint32_t R[16][4];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const uint4 v = *reinterpret_cast<const uint4*>(stage + lane_off + i * row_pitch);
                R[i][0] = v.x; R[i][1] = v.y; R[i][2] = v.z; R[i][3] = v.w;
            }
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                uint32_t x[16], y[16];
#pragma unroll
                for (int i = 0; i < 16; ++i)
                    x[i] = __byte_perm(R[i][m >> 1], 0u, (m & 1) ? 0x4342 : 0x4140);
                net_fwd(x, y);
                // bias both lanes by 2^15 so every lane is a non-negative 16-bit
                // field (|T·X| <= 4080): the byte permute below is then exact.
#pragma unroll
                for (int k = 0; k < 16; ++k) o[m][k] = y[k] + 0x80008000u;
            }
        } else {
            uint32_t R[16][8];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const uint4 a = *reinterpret_cast<const uint4*>(stage + lane_off + i * row_pitch);
                const uint4 b = *reinterpret_cast<const uint4*>(stage + lane_off + i * row_pitch + 16);
                R[i][0] = a.x; R[i][1] = a.y; R[i][2] = a.z; R[i][3] = a.w;
                R[i][4] = b.x; R[i][5] = b.y; R[i][6] = b.z; R[i][7] = b.w;
            }
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                uint32_t x[16], y[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) x[i] = R[i][m];   // int16 pair = SWAR pair
                net_fwd(x, y);
#pragma unroll
                for (int k = 0; k < 16; ++k) o[m][k] = y[k] + 0x80008000u;   // |T·X| <= 16368
            }
        }
        __syncwarp();
        // stage s fully consumed by every lane: refill it with the tile kStages ahead
        if (lane == 0) {
            const long long nt = claims.next();
#pragma unroll
            for (int q = 0; q < kStages; ++q)
                if (q == s) ring[q] = nt;
            if (nt < p.n_tiles) issue_tile<ELEM>(&tin, p, nt, stage, &bars[s], pol);
        }

        // ---- row pass, two rows of Z per step, staged + TMA-stored
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            int32_t z0[16], z1[16];   // rows 2r and 2r+1 of Z
            uint32_t w16[16];         // the same two rows as int16 pairs (store mode 8)
            if constexpr (ELEM == 1) {
                uint32_t x[16], y[16];
#pragma unroll
                for (int m = 0; m < 8; ++m) {
                    x[2 * m] = __byte_perm(o[m][2 * r], o[m][2 * r + 1], 0x5410);
                    x[2 * m + 1] = __byte_perm(o[m][2 * r], o[m][2 * r + 1], 0x7632);
                }
                net_fwd(x, y);
                y[0] -= 0x00080000u;   // remove 16 x (2^15 + 2^31) bias of output l = 0
                if constexpr (SC::kOut16) {
                    // y[l] = Z[2r][l] + 2^16·Z[2r+1][l] (mod 2^32) with the low field in int16
                    // (Z_00 in uint16, no borrow): the int16 rows are the low halves and,
                    // after undoing the borrow, the high halves
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const uint32_t h0 = (r == 0 && q == 0) ? y[0] : y[2 * q] + 0x8000u;
                        const uint32_t h1 = y[2 * q + 1] + 0x8000u;
                        w16[q] = __byte_perm(y[2 * q], y[2 * q + 1], 0x5410);
                        w16[8 + q] = __byte_perm(h0, h1, 0x7632);
                    }
                }
#pragma unroll
                for (int l = 0; l < 16 && !SC::kOut16; ++l) {
                    int32_t lo;
                    if (r == 0 && l == 0) lo = static_cast<int32_t>(y[l] & 0xFFFFu);   // Z_00 in [0, 65280]
                    else lo = static_cast<int32_t>(static_cast<int16_t>(y[l] & 0xFFFFu));
                    z0[l] = lo;
                    z1[l] = static_cast<int32_t>(y[l] - static_cast<uint32_t>(lo)) >> 16;
                }
            } else {
                int32_t x0[16], x1[16];
#pragma unroll
                for (int m = 0; m < 8; ++m) {
                    x0[2 * m] = static_cast<int32_t>(o[m][2 * r] & 0xFFFFu);
                    x0[2 * m + 1] = static_cast<int32_t>(o[m][2 * r] >> 16);
                    x1[2 * m] = static_cast<int32_t>(o[m][2 * r + 1] & 0xFFFFu);
                    x1[2 * m + 1] = static_cast<int32_t>(o[m][2 * r + 1] >> 16);
                }
                net_fwd(x0, z0);
                net_fwd(x1, z1);
                z0[0] -= 16 * 32768;   // inputs carried a +2^15 bias
                z1[0] -= 16 * 32768;
            }
            const int half = r % SC::kPairs;   // position of this row pair inside its store
            if (half == 0 && SM != 2) {
                // the buffer about to be reused must have been read by its TMA store
                if (lane == 0) bulk_wait_read<SC::kBufs - 1>();
            }
            __syncwarp();
            uint8_t* buf = outb + obuf * SC::kBytes;
            if constexpr (SC::kOut16) {
                // staging row (64 B) of this lane inside the box {32 int16, box_b blocks, 8}:
                // 64-byte swizzle, chunk ^= (address >> 7) & 3
                uint8_t* ob = buf + (half * box_b + lane) * 64;
                const int sw = (smem_addr(ob) >> 7) & 3;
                if (lane < box_b) {
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        *reinterpret_cast<uint4*>(ob + ((c ^ sw) << 4)) =
                            make_uint4(w16[4 * c], w16[4 * c + 1], w16[4 * c + 2], w16[4 * c + 3]);
                }
            }
            // staging row of this lane inside the TMA box {32 ints, box_b blocks, kPairs}
            uint8_t* ob = buf + (half * box_b + lane) * 128;
            const int sw = (smem_addr(ob) >> 7) & 7;   // 128-byte swizzle: chunk ^= row & 7
            if (!SC::kOut16 && (SM == 2 || lane < box_b)) {
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    *reinterpret_cast<int4*>(ob + ((c ^ sw) << 4)) =
                        make_int4(z0[4 * c], z0[4 * c + 1], z0[4 * c + 2], z0[4 * c + 3]);
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    *reinterpret_cast<int4*>(ob + (((c + 4) ^ sw) << 4)) =
                        make_int4(z1[4 * c], z1[4 * c + 1], z1[4 * c + 2], z1[4 * c + 3]);
            }
            if constexpr (SM == 2) {
                __syncwarp();
                // lanes 8j..8j+7 move the 128 B row pair of block 4i+j: one warp
                // instruction writes four full 128-byte lines
                const uint8_t* src = buf + (lane >> 3) * 128;
                const int s0 = ((lane & 7) ^ (lane >> 3)) << 4, s1 = ((lane & 7) ^ (4 + (lane >> 3))) << 4;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int4 v = *reinterpret_cast<const int4*>(src + i * 512 + ((i & 1) ? s1 : s0));
                    if (4 * i + (lane >> 3) < nvalid) __stcs(tile_dst + i * 256 + r * 8, v);
                }
                __syncwarp();
            } else if (half == SC::kPairs - 1) {
                fence_async_smem();
                __syncwarp();
                if (lane == 0) {
                    tma_store_4d(&tout, buf, 0, bx0, r - half,
                                 static_cast<int32_t>(strip));
                    bulk_commit();
                }
                obuf = obuf + 1 == SC::kBufs ? 0 : obuf + 1;
            }
        }
    }
    if (lane == 0) {
        bulk_wait<0>();
        claims_done(sched, p.total_warps);   // every warp has claimed past the end
    }
}

namespace {

template <int ELEM, int SM>
int launch_fwd_t(const void* src, const Geom& g, int32_t* coef, cudaStream_t st) {
    using Cfg = FwdCfg<ELEM, SM>;
    CUtensorMap tin, tout;
    const int box_w = g.W < 256 ? g.W : 256;
    {
        const uint64_t dims[3] = {uint64_t(g.W), uint64_t(g.H), uint64_t(g.N)};
        const uint64_t strides[2] = {uint64_t(g.pitch), uint64_t(g.istride)};
        const uint32_t box[3] = {uint32_t(box_w), 16u, 1u};
        int rc = encode_tiled(&tin, ELEM == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_UINT16,
                              3, src, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
        if (rc) return DCT16A_ECUDA;
    }
    if (StoreCfg<SM>::kOut16) {
        // int16 coef viewed as {32 int16 of a row pair, block column bx, row pair, strip}
        const uint64_t dims[4] = {32u, uint64_t(g.BX), 8u, uint64_t(g.N) * uint64_t(g.BY)};
        const uint64_t strides[3] = {512u, 64u, uint64_t(g.BX) * 512u};
        const uint32_t box[4] = {32u, uint32_t(g.BX < 32 ? g.BX : 32), 8u, 1u};
        int rc = encode_tiled(&tout, CU_TENSOR_MAP_DATA_TYPE_UINT16, 4, coef, dims, strides, box,
                              CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE);
        if (rc) return DCT16A_ECUDA;
    } else {
        // coef viewed as {32 int32 of a row pair, block column bx, row pair, strip}
        const uint64_t dims[4] = {32u, uint64_t(g.BX), 8u, uint64_t(g.N) * uint64_t(g.BY)};
        const uint64_t strides[3] = {1024u, 128u, uint64_t(g.BX) * 1024u};
        const uint32_t box[4] = {32u, uint32_t(g.BX < 32 ? g.BX : 32), uint32_t(StoreCfg<SM>::kPairs), 1u};
        int rc = encode_tiled(&tout, CU_TENSOR_MAP_DATA_TYPE_INT32, 4, coef, dims, strides, box,
                              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE);
        if (rc) return DCT16A_ECUDA;
    }
    FwdParams p;
    p.W = g.W;
    p.BX = g.BX;
    p.BY = g.BY;
    p.tiles_per_strip = (g.BX + kTile - 1) / kTile;
    p.box_w = box_w;
    p.n_tiles = static_cast<long long>(g.N) * g.BY * p.tiles_per_strip;

    if (int e = smem_optin(reinterpret_cast<const void*>(fwd_kernel<ELEM, SM>), Cfg::kSmem)) return e;
    const long long want = (p.n_tiles + Cfg::kWarps - 1) / Cfg::kWarps;
    long long grid = static_cast<long long>(num_sms()) * Cfg::kMinCtas;
    if (want < grid) grid = want;
    p.total_warps = static_cast<int>(grid) * Cfg::kWarps;
    SchedGuard guard(kSchedForward, st);
    if (guard.error()) return guard.error();
    p.slot = guard.slot();
    fwd_kernel<ELEM, SM><<<static_cast<unsigned>(grid), Cfg::kWarps * 32, Cfg::kSmem, st>>>(tin, tout, coef, p);
    return static_cast<int>(cudaGetLastError());
}

// Output path of the forward kernel.  Default (8-bit): one 32 KB TMA tensor
// store of the whole tile (mode 5), measured fastest on config 2 with the
// dynamic tile scheduler (6.72 TB/s); 10-bit: 8 KB stores
// (mode 3, 6.68 TB/s on 200 config-4 frames, tools/fwd10_modes.py); the option DCT16A_OPT_FWD_STORE (include/dct16a.h) selects
// the other variants for experiments (profiles/r01_fwd_store_modes.md).
int store_mode(int elem) {
    const int m = get_option(DCT16A_OPT_FWD_STORE);
    return m >= 0 ? m : (elem == 1 ? 5 : 3);
}

template <int ELEM>
int launch_fwd_e(const void* src, const Geom& g, int32_t* coef, cudaStream_t st) {
    switch (store_mode(ELEM)) {
        case 3: return launch_fwd_t<ELEM, 3>(src, g, coef, st);
        case 5: return launch_fwd_t<ELEM, 5>(src, g, coef, st);
#ifdef DCT16A_EXPERIMENTS
        // the store-path experiments of profiles/r01_fwd_store_modes.md (tools/variants.py)
        case 0: return launch_fwd_t<ELEM, 0>(src, g, coef, st);
        case 1: return launch_fwd_t<ELEM, 1>(src, g, coef, st);
        case 2: return launch_fwd_t<ELEM, 2>(src, g, coef, st);
        case 4: return launch_fwd_t<ELEM, 4>(src, g, coef, st);
        case 6: return launch_fwd_t<ELEM, 6>(src, g, coef, st);
        case 7: return launch_fwd_t<ELEM, 7>(src, g, coef, st);
#endif
        default: return DCT16A_EDOMAIN;   // dct16a_set_option admits only the built modes
    }
}

}  // namespace

int launch_forward(const void* src, const Geom& g, int32_t* coef, cudaStream_t st) {
    return g.elem == 1 ? launch_fwd_e<1>(src, g, coef, st) : launch_fwd_e<2>(src, g, coef, st);
}

// 16-bit coefficients, 8-bit images only (every Z fits 16 bits: AC in int16,
// Z_00 in [0, 65280] as uint16 — SURVEY V9, next item f4)
int launch_forward16(const void* src, const Geom& g, int16_t* coef, cudaStream_t st) {
    return launch_fwd_t<1, 8>(src, g, reinterpret_cast<int32_t*>(coef), st);
}

}  // namespace dct16a
