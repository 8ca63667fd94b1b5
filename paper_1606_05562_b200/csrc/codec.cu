// codec.cu — K4 quantize, K5 inverse, K6 SSE/PSNR and the generic fused codec
// (forward -> quantise -> inverse -> reconstruct -> SSE) of the §4 pipeline,
// PAPER.md:866-910, with S folded into the quantiser.
// Exactness rules: quant.cuh.
//
// Generic fused codec layout (zonal, any r, 8- or 10-bit): one warp owns a
// pair of horizontally adjacent blocks (lanes 0-15: block 2px, lanes 16-31:
// block 2px+1), one lane per row/column; persistent CTAs walk a contiguous range
// of block pairs so the per-image SSE is accumulated in registers and flushed
// with one atomic per warp and image.  Both in-block transpositions (the
// paper's transposition buffer) go through a per-warp smem
// tile; per-lane constants (weights, mask, float64 scale factors) are computed
// once per thread.
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include <type_traits>

#include "internal.h"
#include "net16.cuh"
#include "ptx.cuh"
#include "quant.cuh"
#include "tables.cuh"
#include "uexact.cuh"

namespace dct16a {

// ------------------------------------------------------------------ K4
// Elementwise over int4 groups of coefficients.  The grid stride is a multiple
// of 64 int4 (one 16x16 block), so every thread always sees the same four
// cells (k, l0..l0+3): their zig-zag mask, scale s_k·s_l and exact-decision
// constants are computed once per thread.  Streaming loads/stores (.cs).
constexpr int kQUnroll = 4;   // int4 groups in flight per thread

__global__ void __launch_bounds__(256) quantize_kernel(const int4* __restrict__ coef, int4* __restrict__ qcoef,
                                                       float4* __restrict__ scaled, long long n4, long long chunk,
                                                       int mode, int r, int step) {
    // CTA b owns the contiguous int4 range [b·chunk, (b+1)·chunk) (chunk a multiple
    // of 256·kQUnroll), walked kQUnroll·256 int4 at a time with every load of a
    // round issued before any store: a compact address window per CTA, several
    // 16-byte loads in flight per thread
    const long long base = blockIdx.x * chunk;
    const long long lim = min(base + chunk, n4);
    const int pos = static_cast<int>((threadIdx.x * 4) & 255);   // the same 4 cells on every visit
    const int k = pos >> 4, l0 = pos & 15;
    float sc[4], cq[4];
    uint64_t d2g[4];
    bool keep[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const int l = l0 + e;
        const double s = s_of(k) * s_of(l);
        sc[e] = static_cast<float>(s);
        cq[e] = static_cast<float>(s / step);
        d2g[e] = static_cast<uint64_t>(step) * step * (g_of(k) * g_of(l));
        keep[e] = zigzag_rank(k, l) < r;
    }
    for (long long i0 = base + threadIdx.x; i0 < lim; i0 += 256 * kQUnroll) {
        int4 z[kQUnroll];
#pragma unroll
        for (int u = 0; u < kQUnroll; ++u) {
            const long long i = i0 + 256LL * u;
            z[u] = i < lim ? __ldcs(coef + i) : make_int4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < kQUnroll; ++u) {
            const long long i = i0 + 256LL * u;
            if (i >= lim) break;
            int4 q;
            if (mode == DCT16A_ZONAL) {
                q = make_int4(keep[0] ? z[u].x : 0, keep[1] ? z[u].y : 0, keep[2] ? z[u].z : 0, keep[3] ? z[u].w : 0);
            } else {
                q = make_int4(uniform_level(z[u].x, cq[0], d2g[0]), uniform_level(z[u].y, cq[1], d2g[1]),
                              uniform_level(z[u].z, cq[2], d2g[2]), uniform_level(z[u].w, cq[3], d2g[3]));
            }
            __stcs(qcoef + i, q);
            if (scaled) {
                // zonal: s_k·s_l·(Z ⊙ M_r); uniform: s_k·s_l·Z
                const int4 v = mode == DCT16A_ZONAL ? q : z[u];
                __stcs(scaled + i, make_float4(sc[0] * static_cast<float>(v.x), sc[1] * static_cast<float>(v.y),
                                               sc[2] * static_cast<float>(v.z), sc[3] * static_cast<float>(v.w)));
            }
        }
    }
}

namespace {

#ifdef DCT16A_EXPERIMENTS   // the generic codec kernel reads rows straight from global memory
__device__ __forceinline__ void load_row(const uint8_t* p, int elem, int32_t (&x)[16]) {
    if (elem == 1) {
        const uint4 v = __ldcs(reinterpret_cast<const uint4*>(p));
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int j = 0; j < 16; ++j) x[j] = (w[j >> 2] >> (8 * (j & 3))) & 0xFF;
    } else {
        const uint4 a = __ldcs(reinterpret_cast<const uint4*>(p));
        const uint4 b = __ldcs(reinterpret_cast<const uint4*>(p + 16));
        const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
        for (int j = 0; j < 16; ++j) x[j] = static_cast<int16_t>((w[j >> 1] >> (16 * (j & 1))) & 0xFFFF);
    }
}
#endif

__device__ __forceinline__ void store_row(uint8_t* p, int elem, const int (&v)[16]) {
    if (elem == 1) {
        uint32_t w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
            w[q] = __byte_perm(__byte_perm(v[4 * q], v[4 * q + 1], 0x0040), __byte_perm(v[4 * q + 2], v[4 * q + 3], 0x0040),
                               0x5410);
        __stcs(reinterpret_cast<uint4*>(p), make_uint4(w[0], w[1], w[2], w[3]));
    } else {
        uint32_t w[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) w[q] = __byte_perm(v[2 * q], v[2 * q + 1], 0x5410);
        __stcs(reinterpret_cast<uint4*>(p), make_uint4(w[0], w[1], w[2], w[3]));
        __stcs(reinterpret_cast<uint4*>(p + 16), make_uint4(w[4], w[5], w[6], w[7]));
    }
}

// 64-bit block index -> byte offset of its top-left pixel and image index
__device__ __forceinline__ long long block_offset(long long b, const Geom& g, int* n_out, int* row0_out) {
    const long long per_img = static_cast<long long>(g.BY) * g.BX;
    const int n = static_cast<int>(b / per_img);
    const int rem = static_cast<int>(b - n * per_img);
    const int by = rem / g.BX;
    const int bx = rem - by * g.BX;
    *n_out = n;
    *row0_out = by * 16;
    return n * g.istride + static_cast<long long>(by * 16) * g.pitch + bx * 16LL * g.elem;
}

}  // namespace

// ------------------------------------------------------------------ K5
// 16 threads per block (thread t: column t, then row t); each warp owns a pair
// of consecutive blocks (2 KB of block-major levels) and works independently:
// its lane 0 streams the warp's next pair into the second of two per-warp smem
// buffers by bulk copies (one per block, slots 16 words apart so the two
// blocks of the warp read different banks) while the current pair computes;
// the in-block transposition is a per-warp smem tile (no CTA barrier).
// Per-thread column constants are computed once.  Zonal: exact int32 networks
// (any int32 levels with |N| < 2^31); uniform: float64 with the exact decision
// near .5 (reading A10).
constexpr int kInvWarps = 4;
constexpr int kInvSlot = 256 + 16;   // words per block slot in a level buffer

template <bool UNIFORM>
__global__ void __launch_bounds__(kInvWarps * 32) inverse_kernel(const int32_t* __restrict__ qcoef, uint8_t* recon,
                                                                 const Geom g, int step) {
    using V = typename std::conditional<UNIFORM, double, int32_t>::type;
    __shared__ V sm[kInvWarps][2][16][17];
    __shared__ __align__(16) int32_t lv[kInvWarps][2][2 * kInvSlot];
    __shared__ __align__(8) uint64_t bars[kInvWarps][2];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int h = lane >> 4, t = lane & 15;
    const int maxpix = (1 << g.bits) - 1;
    // column t constants: zonal W = 2304/(g_k·g_t); uniform Δ·s_k·s_t by class of k
    int32_t wcol[16];
    double wq[3];
#pragma unroll
    for (int k = 0; k < 16; ++k) wcol[k] = w_of(k, t);
#pragma unroll
    for (int c = 0; c < 3; ++c) wq[c] = static_cast<double>(step) * s_of(c == 0 ? 0 : (c == 1 ? 2 : 3)) * s_of(t);
    const long long npairs = (g.nblocks + 1) / 2;
    const long long stride = static_cast<long long>(gridDim.x) * kInvWarps;
    long long pr = static_cast<long long>(blockIdx.x) * kInvWarps + warp;
    uint64_t* bar = bars[warp];
    auto issue = [&](long long pp, int buf) {   // lane 0: the levels of block pair pp
        const int nv = static_cast<int>(min(2LL, g.nblocks - 2 * pp));
        fence_async_smem();   // this warp's generic reads of the buffer (ordered by __syncwarp) precede the copy
        mbar_arrive_expect_tx(&bar[buf], static_cast<uint32_t>(nv * 1024));
        for (int i = 0; i < nv; ++i) bulk_load(&lv[warp][buf][i * kInvSlot], qcoef + (2 * pp + i) * 256, 1024u, &bar[buf]);
    };
    if (lane == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
        if (pr < npairs) issue(pr, 0);
    }
    __syncwarp();
    for (int it = 0; pr < npairs; pr += stride, ++it) {
        const int buf = it & 1;
        // the other buffer was last read in iteration it-1, closed by its final __syncwarp
        if (lane == 0 && pr + stride < npairs) issue(pr + stride, buf ^ 1);
        mbar_wait(&bar[buf], (it >> 1) & 1);
        const long long b = 2 * pr + h;
        const bool valid = b < g.nblocks;
        const int32_t* blk = &lv[warp][buf][h * kInvSlot];
        V (*tile)[17] = sm[warp][h];
        if (valid) {
            // column t of the level block, weighted: c_k = weight(k, t)·qcoef[k][t]
            V c[16], u[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                const int32_t q = blk[k * 16 + t];
                if constexpr (UNIFORM) {
                    const int gk = g_of(k);
                    c[k] = __int2double_rn(q) * wq[gk == 16 ? 0 : (gk == 12 ? 1 : 2)];
                } else {
                    c[k] = q * wcol[k];
                }
            }
            net_inv(c, u);   // Tᵀ applied down the column
#pragma unroll
            for (int i = 0; i < 16; ++i) tile[i][t] = u[i];
        }
        __syncwarp();
        if (valid) {
            V rrow[16], a[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) rrow[j] = tile[t][j];
            net_inv(rrow, a);   // ... and along row t: A′ = Tᵀ·B̂·T
            int pix[16];
            if constexpr (UNIFORM) {
                // floor(A′ + 1/2) from the float64 value; pixels within 2^-20 of a .5
                // boundary are decided exactly from the levels (uexact.cuh, reading A10)
                uint32_t nm = 0;
                int n0[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    bool nr;
                    pix[j] = round_f64(a[j], nr, n0[j]);
                    nm |= (nr ? 1u : 0u) << j;
                }
                if (nm) {
                    int32_t qb[256];
                    for (int i = 0; i < 256; ++i) qb[i] = blk[i];
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        if ((nm >> j) & 1u) pix[j] = uniform_exact_floor(qb, t, j, step, n0[j]);
                }
#pragma unroll
                for (int j = 0; j < 16; ++j) pix[j] = min(max(pix[j], 0), maxpix);
            } else {
#pragma unroll
                for (int j = 0; j < 16; ++j) pix[j] = zonal_pixel(a[j], maxpix);
            }
            int n, row0;
            const long long off = block_offset(b, g, &n, &row0);
            store_row(recon + off + static_cast<long long>(t) * g.pitch, g.elem, pix);
        }
        __syncwarp();   // the tile and lv[buf] are rewritten later
    }
}

#ifdef DCT16A_EXPERIMENTS
// Experiment build only (codec path 1, tools/variants.py).
// ------------------------------------------------------- fused codec (K2/K3)
struct CodecParams {
    int PX;                  // block pairs per strip = ceil(BX / 2)
    long long n_pairs;       // N·BY·PX
    long long chunk;         // pairs per CTA
    int r, step;
};

constexpr int kCodecWarps = 8;   // static smem < 48 KB per CTA

// Generic fused zonal codec (cross-check kernel, option DCT16A_OPT_CODEC_PATH = 1):
// exact int32 throughout, N = Tᵀ·(W ⊙ M_r ⊙ Z)·T and pixel = round(N/2304).
__global__ void __launch_bounds__(kCodecWarps * 32) codec_kernel(const uint8_t* __restrict__ src, uint8_t* recon,
                                                                unsigned long long* sse, const Geom g,
                                                                const CodecParams cp) {
    // per warp: forward transposition tile (int32, row pitch 20 words) and
    // inverse transposition tile (row pitch 17); block 1 offset by a bank shift
    __shared__ __align__(16) int32_t sy[kCodecWarps][2][16 * 20 + 16];
    __shared__ int32_t su[kCodecWarps][2][16][17];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int h = lane >> 4, t = lane & 15;
    int32_t* ty = &sy[warp][h][h * 16];
    int32_t(*tu)[17] = su[warp][h];

    // per-lane weights of column t (lane = column in the column pass): W ⊙ M_r
    int32_t wcol[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) wcol[k] = zigzag_rank(k, t) < cp.r ? w_of(k, t) : 0;
    const int maxpix = (1 << g.bits) - 1;
    const long long p0 = static_cast<long long>(blockIdx.x) * cp.chunk;
    long long p1 = p0 + cp.chunk;
    if (p1 > cp.n_pairs) p1 = cp.n_pairs;
    // decode the first pair of this warp; later pairs advance incrementally
    long long p = p0 + warp;
    const long long strips = p / cp.PX;
    int px = static_cast<int>(p - strips * cp.PX);
    int n = static_cast<int>(strips / g.BY);
    int by = static_cast<int>(strips - static_cast<long long>(n) * g.BY);
    int cur_n = n;
    unsigned long long acc = 0;

    for (; p < p1; p += kCodecWarps) {
        const int bx = 2 * px + h;
        const bool valid = bx < g.BX;
        const long long off = n * g.istride + static_cast<long long>(by * 16 + t) * g.pitch + bx * 16LL * g.elem;
        if (n != cur_n) {   // image changed (warp-uniform): flush the SSE of the previous one
#pragma unroll
            for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (lane == 0 && acc) atomicAdd(sse + cur_n, acc);
            acc = 0;
            cur_n = n;
        }
        // ---- row t of X, row pass of the forward transform: Y = X·Tᵀ
        int32_t x[16];
        if (valid) load_row(src + off, g.elem, x);
        else {
#pragma unroll
            for (int j = 0; j < 16; ++j) x[j] = 0;
        }
        {
            int32_t y[16];
            net_fwd(x, y);
#pragma unroll
            for (int q = 0; q < 4; ++q)
                *reinterpret_cast<int4*>(ty + t * 20 + 4 * q) = make_int4(y[4 * q], y[4 * q + 1], y[4 * q + 2], y[4 * q + 3]);
        }
        __syncwarp();
        // ---- column t: Z[:, t] = T·Y[:, t]; quantise; inverse down the column
        {
            int32_t col[16], z[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) col[k] = ty[k * 20 + t];
            net_fwd(col, z);
            int32_t c[16], u[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) c[k] = z[k] * wcol[k];
            net_inv(c, u);
#pragma unroll
            for (int i = 0; i < 16; ++i) tu[i][t] = u[i];
        }
        __syncwarp();
        // ---- row t: A′[t, :] = (Tᵀ·B̂)[t, :]·T, round, clamp, SSE, store
        int32_t rr[16], a[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) rr[j] = tu[t][j];
        net_inv(rr, a);
        int pix[16];
        uint32_t e = 0;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            pix[j] = zonal_pixel(a[j], maxpix);
            const int d = pix[j] - x[j];
            e += static_cast<uint32_t>(d * d);
        }
        if (valid) {
            if (by * 16 + t < g.VH) acc += e;
            if (recon) store_row(recon + off, g.elem, pix);
        }
        __syncwarp();
        // next pair of this warp
        px += kCodecWarps;
        while (px >= cp.PX) {
            px -= cp.PX;
            if (++by == g.BY) {
                by = 0;
                ++n;
            }
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0 && acc) atomicAdd(sse + cur_n, acc);
}

#endif  // DCT16A_EXPERIMENTS

// ------------------------------------------------------------------ K6
__global__ void sse_kernel(const uint8_t* __restrict__ a, const uint8_t* __restrict__ b,
                           unsigned long long* sse, const Geom g) {
    const uint32_t cpr = static_cast<uint32_t>(g.W * g.elem / 16);   // 16-byte chunks per row
    __shared__ uint64_t ws[32];
    for (int n = blockIdx.y; n < g.N; n += gridDim.y) {   // gridDim.y <= 65535: stride over images
    // chunks of one image: VH·cpr < 2^31 (validated by the launcher), so 32-bit index arithmetic
    const uint32_t total = static_cast<uint32_t>(g.VH) * cpr;
    uint64_t acc = 0;
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < total; c += gridDim.x * blockDim.x) {
        const uint32_t row = c / cpr;
        const uint32_t col = c - row * cpr;
        const long long off = n * g.istride + static_cast<long long>(row) * g.pitch + col * 16LL;
        const uint4 va = __ldcs(reinterpret_cast<const uint4*>(a + off));
        const uint4 vb = __ldcs(reinterpret_cast<const uint4*>(b + off));
        const uint32_t wa[4] = {va.x, va.y, va.z, va.w}, wb[4] = {vb.x, vb.y, vb.z, vb.w};
        uint32_t e = 0;   // <= 16·255² (8-bit) or 8·1023² (10-bit): fits 32 bits
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (g.elem == 1) {
                const uint32_t d = __vabsdiffu4(wa[q], wb[q]);   // |x - y| per byte
                e = __dp4a(d, d, e);
            } else {
                const uint32_t d = __vabsdiffu2(wa[q], wb[q]);   // |x - y| per 16-bit pixel (both in [0, 1023])
                const uint32_t lo = d & 0xFFFFu, hi = d >> 16;
                e += lo * lo + hi * hi;
            }
        }
        acc += e;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint64_t s = 0;
        for (int w = 0; w < (blockDim.x >> 5); ++w) s += ws[w];
        if (s) atomicAdd(sse + n, static_cast<unsigned long long>(s));
    }
    __syncthreads();
    }
}

__global__ void psnr_kernel(const unsigned long long* sse, double* psnr, int n, double peak2P) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const unsigned long long s = sse[i];
    psnr[i] = s == 0 ? INFINITY : 10.0 * log10(peak2P / static_cast<double>(s));
}

// PSNR of `count` SSE values of images of geometry g (peak 2^b - 1, P = VH·W).
int launch_psnr_finish(const Geom& g, long long count, uint64_t* sse, double* psnr, cudaStream_t st) {
    if (!psnr) return 0;
    const double peak = static_cast<double>((1 << g.bits) - 1);
    const double P = static_cast<double>(g.VH) * g.W;
    psnr_kernel<<<static_cast<unsigned>((count + 127) / 128), 128, 0, st>>>(reinterpret_cast<unsigned long long*>(sse),
                                                                         psnr, static_cast<int>(count), peak * peak * P);
    return static_cast<int>(cudaGetLastError());
}

// The exact total of `n` SSE values and the PSNR of the whole set (one CTA:
// config 4's global PSNR after the SSE all-reduce, reading A8).
__global__ void __launch_bounds__(1024) sse_total_kernel(const unsigned long long* sse, long long n,
                                                         unsigned long long* total, double* psnr_total,
                                                         double peak2P) {
    __shared__ unsigned long long ws[32];
    unsigned long long acc = 0;
    for (long long i = threadIdx.x; i < n; i += blockDim.x) acc += sse[i];
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long s = 0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) s += ws[w];
        if (total) *total = s;
        if (psnr_total) *psnr_total = s == 0 ? INFINITY : 10.0 * log10(peak2P * static_cast<double>(n) / static_cast<double>(s));
    }
}

int launch_sse_total(const Geom& g, long long count, const uint64_t* sse, uint64_t* total, double* psnr_total,
                     cudaStream_t st) {
    if (!total && !psnr_total) return 0;
    const double peak = static_cast<double>((1 << g.bits) - 1);
    const double P = static_cast<double>(g.VH) * g.W;
    sse_total_kernel<<<1, 1024, 0, st>>>(reinterpret_cast<const unsigned long long*>(sse), count,
                                        reinterpret_cast<unsigned long long*>(total), psnr_total, peak * peak * P);
    return static_cast<int>(cudaGetLastError());
}

namespace {
int finish_psnr(const Geom& g, uint64_t* sse, double* psnr, cudaStream_t st) {
    return launch_psnr_finish(g, g.N, sse, psnr, st);
}
}  // namespace

int launch_quantize(const int32_t* coef, const Geom& g, const dct16a_quant& q, int32_t* qcoef,
                    float* scaled, cudaStream_t st) {
    const long long n4 = g.nblocks * 64;
    const long long per = 256LL * kQUnroll;
    long long grid = static_cast<long long>(num_sms()) * 8;
    long long chunk = (n4 + grid - 1) / grid;
    chunk = (chunk + per - 1) / per * per;   // whole rounds: every thread keeps its 4 cells
    grid = (n4 + chunk - 1) / chunk;
    quantize_kernel<<<static_cast<unsigned>(grid), 256, 0, st>>>(
        reinterpret_cast<const int4*>(coef), reinterpret_cast<int4*>(qcoef), reinterpret_cast<float4*>(scaled),
        n4, chunk, q.mode, q.r, q.step);
    return static_cast<int>(cudaGetLastError());
}

int launch_inverse(const int32_t* qcoef, const Geom& g, const dct16a_quant& q, void* recon, cudaStream_t st) {
    const long long npairs = (g.nblocks + 1) / 2;
    long long grid = (npairs + kInvWarps - 1) / kInvWarps;
    const long long cap = static_cast<long long>(num_sms()) * (q.mode == DCT16A_UNIFORM ? 4 : 8);
    if (grid > cap) grid = cap;
    if (q.mode == DCT16A_UNIFORM)
        inverse_kernel<true><<<static_cast<unsigned>(grid), kInvWarps * 32, 0, st>>>(qcoef, static_cast<uint8_t*>(recon), g, q.step);
    else
        inverse_kernel<false><<<static_cast<unsigned>(grid), kInvWarps * 32, 0, st>>>(qcoef, static_cast<uint8_t*>(recon), g, q.step);
    return static_cast<int>(cudaGetLastError());
}

int launch_psnr(const void* ref, const void* test, const Geom& g, uint64_t* sse, double* psnr, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(sse, 0, sizeof(uint64_t) * g.N, st);
    if (e) return static_cast<int>(e);
    const long long chunks = static_cast<long long>(g.VH) * (g.W * g.elem / 16);
    long long gx = (chunks + 255) / 256;
    if (gx > 64) gx = 64;
    sse_kernel<<<dim3(static_cast<unsigned>(gx), g.N < 65535 ? g.N : 65535), 256, 0, st>>>(
        static_cast<const uint8_t*>(ref), static_cast<const uint8_t*>(test),
        reinterpret_cast<unsigned long long*>(sse), g);
    e = cudaGetLastError();
    if (e) return static_cast<int>(e);
    return finish_psnr(g, sse, psnr, st);
}

#ifdef DCT16A_EXPERIMENTS
int launch_codec_generic(const void* src, const Geom& g, const dct16a_quant& q, void* recon, uint64_t* sse,
                         cudaStream_t st) {
    CodecParams cp;
    cp.PX = (g.BX + 1) / 2;
    cp.n_pairs = static_cast<long long>(g.N) * g.BY * cp.PX;
    const int ctas_per_sm = 16 / kCodecWarps;
    long long grid = static_cast<long long>(num_sms()) * ctas_per_sm;
    const long long min_chunk = 4 * kCodecWarps;
    if (grid * min_chunk > cp.n_pairs) grid = (cp.n_pairs + min_chunk - 1) / min_chunk;
    cp.chunk = (cp.n_pairs + grid - 1) / grid;
    cp.r = q.r;
    cp.step = q.step;
    codec_kernel<<<static_cast<unsigned>(grid), kCodecWarps * 32, 0, st>>>(
        static_cast<const uint8_t*>(src), static_cast<uint8_t*>(recon), reinterpret_cast<unsigned long long*>(sse), g,
        cp);
    return static_cast<int>(cudaGetLastError());
}
#endif  // DCT16A_EXPERIMENTS

// Kernel choice of the fused codec (option DCT16A_OPT_CODEC_PATH, include/dct16a.h):
//   0 auto: zonal (8/10-bit, every r) -> band-pruned warp-per-tile kernel
//           (zonal_band.cu), uniform -> warp-per-block-pair kernel (codec_warp.cu);
//   2: always codec_warp.cu.
// Experiment builds (-DDCT16A_EXPERIMENTS) add 1 (zonal on the generic kernel
// above), 3 (zonal 8-bit r <= 36 on the thread-per-block kernel, zonal_tpb.cu)
// and 4 (uniform on the two-blocks-per-lane kernel, codec_uniform.cu).  Every
// path computes the same bytes.
int launch_codec(const void* src, const Geom& g, const dct16a_quant& q, void* recon, uint64_t* sse,
                 double* psnr, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(sse, 0, sizeof(uint64_t) * g.N, st);
    if (e) return static_cast<int>(e);
    const int path = get_option(DCT16A_OPT_CODEC_PATH);
    const bool zonal = q.mode == DCT16A_ZONAL;
    int rc;
    if (zonal && path == 0 && zonal_band_applies(g, q.r)) rc = launch_zonal_band(src, g, q.r, recon, sse, st);
#ifdef DCT16A_EXPERIMENTS
    else if (zonal && path == 3 && g.elem == 1 && zonal_band(q.r) <= 7) rc = launch_zonal_tpb(src, g, q.r, recon, sse, st);
    else if (zonal && path == 1) rc = launch_codec_generic(src, g, q, recon, sse, st);
#endif
#ifdef DCT16A_EXPERIMENTS
    else if (!zonal && path == 4) rc = launch_codec_uniform(src, g, q, recon, sse, st, nullptr, 0, 0, 0);
#endif
    else rc = launch_codec_warp(src, g, q, recon, sse, st);
    if (rc) return rc;
    return finish_psnr(g, sse, psnr, st);
}

}  // namespace dct16a
