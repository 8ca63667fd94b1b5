// codec.cu — K4 quantize, K5 inverse, K6 SSE/PSNR and the fused codec
// (forward -> quantise -> inverse -> reconstruct -> SSE) of the §4 pipeline,
// PAPER.md:866-910, with S folded into the quantiser.
//
// Exactness (readings A6, A9, A10):
//  * zonal: N = Tᵀ·(W ⊙ Z ⊙ M_r)·T in int32 (|N| <= 7612·maxpix < 2^24),
//    pixel = clamp(round_half_away(N / 2304)) decided on the integer N;
//  * uniform: q = sign(Z)·m with m the largest integer such that
//    (2m-1)²·Δ²·G <= 4·Z² (G = g_k·g_l), i.e. floor(|Z|/(Δ·sqrt G) + 1/2) with
//    ties away from zero, decided in int64 after a float64 estimate;
//    reconstruction Tᵀ·(Δ·q·s_k·s_l)·T in float64.
#include <math.h>
#include <type_traits>
#include <stdint.h>

#include "internal.h"
#include "net16.cuh"
#include "tables.cuh"

namespace dct16a {
namespace {

__device__ __forceinline__ double inv_sqrt_G(int k, int l) {
    return 1.0 / sqrt(static_cast<double>(g_of(k) * g_of(l)));
}

// exact uniform level (reading A9): floor(|Z|/(step·sqrt(G)) + 1/2), ties away
__device__ __forceinline__ int32_t uniform_level(int32_t z, int k, int l, int step) {
    const int64_t G = g_of(k) * g_of(l);
    const int64_t az = z < 0 ? -static_cast<int64_t>(z) : static_cast<int64_t>(z);
    const double est = static_cast<double>(az) * inv_sqrt_G(k, l) / static_cast<double>(step) + 0.5;
    int64_t m = static_cast<int64_t>(floor(est));
    const int64_t z4 = 4 * az * az;
    const int64_t d2g = static_cast<int64_t>(step) * step * G;
    if (m > 0 && (2 * m - 1) * (2 * m - 1) * d2g > z4) --m;
    else if ((2 * m + 1) * (2 * m + 1) * d2g <= z4) ++m;
    return static_cast<int32_t>(z < 0 ? -m : m);
}

__device__ __forceinline__ int zonal_pixel(int32_t N, int maxpix) {
    // round half away of N/2304, clamped to [0, maxpix] (reading A6)
    const int32_t v = N + 1152;
    if (v <= 0) return 0;
    const int32_t p = v / 2304;
    return p > maxpix ? maxpix : p;
}

__device__ __forceinline__ int uniform_pixel(double a, int maxpix) {
    if (!(a > 0.0)) return 0;            // round_half_away(a) <= 0 -> clamp 0
    const double p = floor(a + 0.5);
    return p > maxpix ? maxpix : static_cast<int>(p);
}

// ------------------------------------------------------------------ K4
}  // namespace

__global__ void quantize_kernel(const int4* __restrict__ coef, int4* __restrict__ qcoef,
                                float4* __restrict__ scaled, long long n4, int mode, int r,
                                int step) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n4;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int4 z = coef[i];
        const int pos = static_cast<int>((i * 4) & 255);
        const int k = pos >> 4, l0 = pos & 15;
        int zz[4] = {z.x, z.y, z.z, z.w};
        int qq[4];
        float ss[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int l = l0 + e;
            const double s = inv_sqrt_G(k, l);
            if (mode == DCT16A_ZONAL) {
                qq[e] = zigzag_rank(k, l) < r ? zz[e] : 0;
                ss[e] = static_cast<float>(s * static_cast<double>(qq[e]));
            } else {
                qq[e] = uniform_level(zz[e], k, l, step);
                ss[e] = static_cast<float>(s * static_cast<double>(zz[e]));
            }
        }
        qcoef[i] = make_int4(qq[0], qq[1], qq[2], qq[3]);
        if (scaled) scaled[i] = make_float4(ss[0], ss[1], ss[2], ss[3]);
    }
}

namespace {
// ------------------------------------------------ block addressing helpers
struct BlkAddr {
    long long img_off;  // byte offset of the block's top-left pixel
    int n, row0;
};

__device__ __forceinline__ BlkAddr block_addr(long long b, const Geom& g) {
    const long long per_img = static_cast<long long>(g.BY) * g.BX;
    BlkAddr a;
    a.n = static_cast<int>(b / per_img);
    const long long rem = b - a.n * per_img;
    const int by = static_cast<int>(rem / g.BX);
    const int bx = static_cast<int>(rem - static_cast<long long>(by) * g.BX);
    a.row0 = by * 16;
    a.img_off = a.n * g.istride + static_cast<long long>(a.row0) * g.pitch + bx * 16LL * g.elem;
    return a;
}

__device__ __forceinline__ void load_row(const uint8_t* p, int elem, int32_t (&x)[16]) {
    if (elem == 1) {
        const uint4 v = *reinterpret_cast<const uint4*>(p);
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int j = 0; j < 16; ++j) x[j] = (w[j >> 2] >> (8 * (j & 3))) & 0xFF;
    } else {
        const uint4 a = *reinterpret_cast<const uint4*>(p);
        const uint4 b = *reinterpret_cast<const uint4*>(p + 16);
        const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
        for (int j = 0; j < 16; ++j) x[j] = static_cast<int16_t>((w[j >> 1] >> (16 * (j & 1))) & 0xFFFF);
    }
}

__device__ __forceinline__ void store_row(uint8_t* p, int elem, const int (&v)[16]) {
    if (elem == 1) {
        uint32_t w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
            w[q] = (v[4 * q] & 0xFF) | ((v[4 * q + 1] & 0xFF) << 8) | ((v[4 * q + 2] & 0xFF) << 16) |
                   (static_cast<uint32_t>(v[4 * q + 3] & 0xFF) << 24);
        *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
    } else {
        uint32_t w[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) w[q] = (v[2 * q] & 0xFFFF) | (static_cast<uint32_t>(v[2 * q + 1] & 0xFFFF) << 16);
        *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
        *reinterpret_cast<uint4*>(p + 16) = make_uint4(w[4], w[5], w[6], w[7]);
    }
}

constexpr int kBlkPerCta = 8;  // 16 threads per block, 128 threads per CTA
}  // namespace

// ------------------------------------------------------------------ K5
template <bool UNIFORM>
__global__ void __launch_bounds__(128) inverse_kernel(const int32_t* __restrict__ qcoef, uint8_t* recon,
                                                      const Geom g, int step) {
    using V = typename std::conditional<UNIFORM, double, int32_t>::type;
    __shared__ V sm[kBlkPerCta][16][17];
    const int sub = threadIdx.x >> 4, t = threadIdx.x & 15;
    const long long b = static_cast<long long>(blockIdx.x) * kBlkPerCta + sub;
    const bool valid = b < g.nblocks;
    if (valid) {
        // column t of the coefficient block: c_k = weight(k, t)·qcoef[k][t]
        V c[16], u[16];
        const int32_t* blk = qcoef + b * 256;
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const int32_t q = blk[k * 16 + t];
            if constexpr (UNIFORM) c[k] = static_cast<double>(step) * static_cast<double>(q) * inv_sqrt_G(k, t);
            else c[k] = q * w_of(k, t);
        }
        net_inv(c, u);   // Tᵀ applied down the column
#pragma unroll
        for (int i = 0; i < 16; ++i) sm[sub][i][t] = u[i];
    }
    __syncthreads();
    if (!valid) return;
    V rrow[16], a[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) rrow[j] = sm[sub][t][j];
    net_inv(rrow, a);    // ... and along row t: A′ = Tᵀ·B̂·T
    const int maxpix = (1 << g.bits) - 1;
    int pix[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        if constexpr (UNIFORM) pix[j] = uniform_pixel(a[j], maxpix);
        else pix[j] = zonal_pixel(a[j], maxpix);
    }
    const BlkAddr ad = block_addr(b, g);
    store_row(recon + ad.img_off + static_cast<long long>(t) * g.pitch, g.elem, pix);
}

// ------------------------------------------------------- fused codec (K2/K3)
template <bool UNIFORM>
__global__ void __launch_bounds__(128) codec_kernel(const uint8_t* __restrict__ src, uint8_t* recon,
                                                    unsigned long long* sse, const Geom g, int r, int step) {
    using V = typename std::conditional<UNIFORM, double, int32_t>::type;
    __shared__ int32_t sy[kBlkPerCta][16][17];
    __shared__ V su[kBlkPerCta][16][17];
    const int sub = threadIdx.x >> 4, t = threadIdx.x & 15;
    const long long b = static_cast<long long>(blockIdx.x) * kBlkPerCta + sub;
    const bool valid = b < g.nblocks;
    BlkAddr ad{};
    int32_t x[16];
    if (valid) {
        ad = block_addr(b, g);
        load_row(src + ad.img_off + static_cast<long long>(t) * g.pitch, g.elem, x);
        int32_t y[16];
        net_fwd(x, y);   // row t of X·Tᵀ
#pragma unroll
        for (int l = 0; l < 16; ++l) sy[sub][t][l] = y[l];
    }
    __syncthreads();
    if (valid) {
        int32_t col[16], z[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) col[i] = sy[sub][i][t];
        net_fwd(col, z);   // column t of Z = T·X·Tᵀ
        V c[16], u[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            if constexpr (UNIFORM)
                c[k] = static_cast<double>(step) * static_cast<double>(uniform_level(z[k], k, t, step)) *
                       inv_sqrt_G(k, t);
            else c[k] = zigzag_rank(k, t) < r ? z[k] * w_of(k, t) : 0;
        }
        net_inv(c, u);
#pragma unroll
        for (int i = 0; i < 16; ++i) su[sub][i][t] = u[i];
    }
    __syncthreads();
    if (!valid) return;
    V rrow[16], a[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) rrow[j] = su[sub][t][j];
    net_inv(rrow, a);
    const int maxpix = (1 << g.bits) - 1;
    int pix[16];
    uint32_t e = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        if constexpr (UNIFORM) pix[j] = uniform_pixel(a[j], maxpix);
        else pix[j] = zonal_pixel(a[j], maxpix);
        const int d = pix[j] - x[j];
        e += static_cast<uint32_t>(d * d);
    }
    if (ad.row0 + t >= g.VH) e = 0;   // rows beyond valid_height do not count
    if (recon) store_row(recon + ad.img_off + static_cast<long long>(t) * g.pitch, g.elem, pix);
#pragma unroll
    for (int o = 8; o; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
    if (t == 0 && e) atomicAdd(sse + ad.n, static_cast<unsigned long long>(e));
}

// ------------------------------------------------------------------ K6
__global__ void sse_kernel(const uint8_t* __restrict__ a, const uint8_t* __restrict__ b,
                           unsigned long long* sse, const Geom g) {
    const int n = blockIdx.y;
    const int cpr = g.W * g.elem / 16;   // 16-byte chunks per row
    const long long total = static_cast<long long>(g.VH) * cpr;
    uint64_t acc = 0;
    for (long long c = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; c < total;
         c += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long row = c / cpr;
        const int col = static_cast<int>(c - row * cpr);
        const long long off = n * g.istride + row * g.pitch + col * 16LL;
        const uint4 va = *reinterpret_cast<const uint4*>(a + off);
        const uint4 vb = *reinterpret_cast<const uint4*>(b + off);
        const uint32_t wa[4] = {va.x, va.y, va.z, va.w}, wb[4] = {vb.x, vb.y, vb.z, vb.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (g.elem == 1) {
#pragma unroll
                for (int s = 0; s < 4; ++s) {
                    const int d = static_cast<int>((wa[q] >> (8 * s)) & 0xFF) - static_cast<int>((wb[q] >> (8 * s)) & 0xFF);
                    acc += static_cast<uint32_t>(d * d);
                }
            } else {
#pragma unroll
                for (int s = 0; s < 2; ++s) {
                    const int d = static_cast<int>(static_cast<int16_t>((wa[q] >> (16 * s)) & 0xFFFF)) -
                                  static_cast<int>(static_cast<int16_t>((wb[q] >> (16 * s)) & 0xFFFF));
                    acc += static_cast<uint64_t>(static_cast<int64_t>(d) * d);
                }
            }
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    __shared__ uint64_t ws[32];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint64_t s = 0;
        for (int w = 0; w < (blockDim.x >> 5); ++w) s += ws[w];
        if (s) atomicAdd(sse + n, static_cast<unsigned long long>(s));
    }
}

__global__ void psnr_kernel(const unsigned long long* sse, double* psnr, int n, double peak2P) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const unsigned long long s = sse[i];
    psnr[i] = s == 0 ? INFINITY : 10.0 * log10(peak2P / static_cast<double>(s));
}

namespace {
int finish_psnr(const Geom& g, uint64_t* sse, double* psnr, cudaStream_t st) {
    if (!psnr) return 0;
    const double peak = static_cast<double>((1 << g.bits) - 1);
    const double P = static_cast<double>(g.VH) * g.W;
    psnr_kernel<<<(g.N + 127) / 128, 128, 0, st>>>(reinterpret_cast<unsigned long long*>(sse), psnr, g.N,
                                                  peak * peak * P);
    return static_cast<int>(cudaGetLastError());
}

}  // namespace

int launch_quantize(const int32_t* coef, const Geom& g, const dct16a_quant& q, int32_t* qcoef,
                    float* scaled, cudaStream_t st) {
    const long long n4 = g.nblocks * 64;
    long long grid = (n4 + 255) / 256;
    const long long cap = static_cast<long long>(num_sms()) * 8;
    if (grid > cap) grid = cap;
    quantize_kernel<<<static_cast<unsigned>(grid), 256, 0, st>>>(
        reinterpret_cast<const int4*>(coef), reinterpret_cast<int4*>(qcoef), reinterpret_cast<float4*>(scaled),
        n4, q.mode, q.r, q.step);
    return static_cast<int>(cudaGetLastError());
}

int launch_inverse(const int32_t* qcoef, const Geom& g, const dct16a_quant& q, void* recon, cudaStream_t st) {
    const long long grid = (g.nblocks + kBlkPerCta - 1) / kBlkPerCta;
    if (q.mode == DCT16A_UNIFORM)
        inverse_kernel<true><<<static_cast<unsigned>(grid), 128, 0, st>>>(qcoef, static_cast<uint8_t*>(recon), g, q.step);
    else
        inverse_kernel<false><<<static_cast<unsigned>(grid), 128, 0, st>>>(qcoef, static_cast<uint8_t*>(recon), g, q.step);
    return static_cast<int>(cudaGetLastError());
}

int launch_psnr(const void* ref, const void* test, const Geom& g, uint64_t* sse, double* psnr, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(sse, 0, sizeof(uint64_t) * g.N, st);
    if (e) return static_cast<int>(e);
    const long long chunks = static_cast<long long>(g.VH) * (g.W * g.elem / 16);
    long long gx = (chunks + 255) / 256;
    if (gx > 64) gx = 64;
    sse_kernel<<<dim3(static_cast<unsigned>(gx), g.N), 256, 0, st>>>(
        static_cast<const uint8_t*>(ref), static_cast<const uint8_t*>(test),
        reinterpret_cast<unsigned long long*>(sse), g);
    e = cudaGetLastError();
    if (e) return static_cast<int>(e);
    return finish_psnr(g, sse, psnr, st);
}

int launch_codec(const void* src, const Geom& g, const dct16a_quant& q, void* recon, uint64_t* sse,
                 double* psnr, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(sse, 0, sizeof(uint64_t) * g.N, st);
    if (e) return static_cast<int>(e);
    const long long grid = (g.nblocks + kBlkPerCta - 1) / kBlkPerCta;
    auto* s = reinterpret_cast<unsigned long long*>(sse);
    if (q.mode == DCT16A_UNIFORM)
        codec_kernel<true><<<static_cast<unsigned>(grid), 128, 0, st>>>(
            static_cast<const uint8_t*>(src), static_cast<uint8_t*>(recon), s, g, q.r, q.step);
    else
        codec_kernel<false><<<static_cast<unsigned>(grid), 128, 0, st>>>(
            static_cast<const uint8_t*>(src), static_cast<uint8_t*>(recon), s, g, q.r, q.step);
    e = cudaGetLastError();
    if (e) return static_cast<int>(e);
    return finish_psnr(g, sse, psnr, st);
}

}  // namespace dct16a
