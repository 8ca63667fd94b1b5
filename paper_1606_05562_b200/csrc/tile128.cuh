// tile128.cuh — the 16-row x 128-pixel tile machinery shared by the
// warp-cooperative kernels (codec_warp.cu, sweep.cu): a tile is 8 horizontally
// adjacent 16x16 blocks of one 16-row strip, brought into shared memory by TMA
// (cp.async.bulk.tensor) as 128-byte-swizzled boxes of 16 rows x 128 bytes
// (one box for uint8, two for uint16), so that the 8 lanes of a quarter-warp
// reading rows 0-7 of one block hit 8 distinct 16-byte chunks.  Every stage
// base must be 1024-byte aligned (the swizzle takes smem address bits 7-9).
// P is any parameter struct with fields W, BY, tiles_per_strip and n_tiles.
#pragma once
#include <cuda.h>
#include <stdint.h>

#include "ptx.cuh"

namespace dct16a {

constexpr int kWTile = 8;     // blocks per tile (128 px)

__device__ __forceinline__ uint8_t* walign1024(uint8_t* smem_raw) {
    return smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
}

// byte offset of the 16-byte chunk c of row t in a 128-byte-swizzled box
__device__ __forceinline__ int swz(int t, int c) { return t * 128 + ((c ^ (t & 7)) << 4); }

template <int ELEM, class P>
__device__ __forceinline__ void w_tile_coords(const P& p, long long tix, int* n, int* by, int* x0) {
    const long long strip = tix / p.tiles_per_strip;
    const int tb = static_cast<int>(tix - strip * p.tiles_per_strip);
    *n = static_cast<int>(strip / p.BY);
    *by = static_cast<int>(strip - static_cast<long long>(*n) * p.BY);
    *x0 = tb * kWTile * 16;
}

// Tile coordinates advanced incrementally (a warp walks a contiguous tile range):
// one division at the start instead of two 64-bit divisions per tile.
struct TileCursor {
    int n, by, tb;
    template <class P>
    __device__ __forceinline__ void init(const P& p, long long tix) {
        if (p.n_tiles <= 0x7FFFFFFFLL) {   // 32-bit divisions (the common case)
            const uint32_t t = static_cast<uint32_t>(tix);
            const uint32_t strip = t / static_cast<uint32_t>(p.tiles_per_strip);
            tb = static_cast<int>(t - strip * static_cast<uint32_t>(p.tiles_per_strip));
            n = static_cast<int>(strip / static_cast<uint32_t>(p.BY));
            by = static_cast<int>(strip - static_cast<uint32_t>(n) * static_cast<uint32_t>(p.BY));
            return;
        }
        int x0;
        w_tile_coords<1>(p, tix, &n, &by, &x0);
        tb = x0 / (kWTile * 16);
    }
    template <class P>
    __device__ __forceinline__ void advance(const P& p) {
        if (++tb == p.tiles_per_strip) {
            tb = 0;
            if (++by == p.BY) {
                by = 0;
                ++n;
            }
        }
    }
    __device__ __forceinline__ int x0() const { return tb * kWTile * 16; }
};

template <int ELEM, class P>
__device__ __forceinline__ void w_issue_at(const CUtensorMap* tin, const P& p, const TileCursor& c, uint8_t* stage,
                                           uint64_t* bar, uint64_t pol) {
    constexpr int box_px = 128 / ELEM;
    const int x0 = c.x0();
    const int nbox = (ELEM == 2 && x0 + box_px < p.W) ? 2 : 1;
    mbar_arrive_expect_tx(bar, static_cast<uint32_t>(nbox * 2048));
    for (int h = 0; h < nbox; ++h) tma_load_3d(stage + h * 2048, tin, bar, x0 + h * box_px, c.by * 16, c.n, pol);
}

template <int ELEM, class P>
__device__ __forceinline__ void w_store_at(const CUtensorMap* tout, const P& p, const TileCursor& c, uint8_t* stage) {
    constexpr int box_px = 128 / ELEM;
    const int x0 = c.x0();
    const int nbox = (ELEM == 2 && x0 + box_px < p.W) ? 2 : 1;
    for (int h = 0; h < nbox; ++h) tma_store_3d(tout, stage + h * 2048, x0 + h * box_px, c.by * 16, c.n);
}

template <int ELEM, class P>
__device__ __forceinline__ void w_issue(const CUtensorMap* tin, const P& p, long long tix, uint8_t* stage,
                                        uint64_t* bar, uint64_t pol) {
    int n, by, x0;
    w_tile_coords<ELEM>(p, tix, &n, &by, &x0);
    constexpr int box_px = 128 / ELEM;
    const int nbox = (ELEM == 2 && x0 + box_px < p.W) ? 2 : 1;
    mbar_arrive_expect_tx(bar, static_cast<uint32_t>(nbox * 2048));
    for (int h = 0; h < nbox; ++h) tma_load_3d(stage + h * 2048, tin, bar, x0 + h * box_px, by * 16, n, pol);
}

template <int ELEM, class P>
__device__ __forceinline__ void w_store(const CUtensorMap* tout, const P& p, long long tix, uint8_t* stage) {
    int n, by, x0;
    w_tile_coords<ELEM>(p, tix, &n, &by, &x0);
    constexpr int box_px = 128 / ELEM;
    const int nbox = (ELEM == 2 && x0 + box_px < p.W) ? 2 : 1;
    for (int h = 0; h < nbox; ++h) tma_store_3d(tout, stage + h * 2048, x0 + h * box_px, by * 16, n);
}

// smem byte offsets (within the stage) of the 16·ELEM bytes of row t of block bb
template <int ELEM>
__device__ __forceinline__ void row_addr(int bb, int t, int* a0, int* a1) {
    if (ELEM == 1) {
        *a0 = swz(t, bb);
        *a1 = *a0;
    } else {
        const int base = (bb >> 2) * 2048, c = (bb & 3) * 2;
        *a0 = base + swz(t, c);
        *a1 = base + swz(t, c + 1);
    }
}

template <int ELEM>
__device__ __forceinline__ void load_px(const uint8_t* stage, int a0, int a1, uint32_t (&w)[4 * ELEM]) {
    const uint4 v = *reinterpret_cast<const uint4*>(stage + a0);
    w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
    if (ELEM == 2) {
        const uint4 u = *reinterpret_cast<const uint4*>(stage + a1);
        w[4] = u.x; w[5] = u.y; w[6] = u.z; w[7] = u.w;
    }
}

// pixel j of a packed row (u8 or u16)
template <int ELEM>
__device__ __forceinline__ int px_of(const uint32_t (&w)[4 * ELEM], int j) {
    return ELEM == 1 ? static_cast<int>((w[j >> 2] >> (8 * (j & 3))) & 0xFFu)
                     : static_cast<int>((w[j >> 1] >> (16 * (j & 1))) & 0xFFFFu);
}

// pixel j of a packed row as float (unsigned extraction: one I2F.U8/U16 with a
// byte / half selector)
template <int ELEM>
__device__ __forceinline__ float px_float(const uint32_t (&w)[4 * ELEM], int j) {
    return ELEM == 1 ? static_cast<float>((w[j >> 2] >> (8 * (j & 3))) & 0xFFu)
                     : static_cast<float>((w[j >> 1] >> (16 * (j & 1))) & 0xFFFFu);
}

}  // namespace dct16a
