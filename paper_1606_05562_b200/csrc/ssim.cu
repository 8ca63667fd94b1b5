// ssim.cu — K9: mean SSIM per image (Wang et al. 2004; the
// parameters are reading A21 of DESIGN.md: 11x11 Gaussian window, sigma 1.5,
// unit sum, K1 = 0.01, K2 = 0.03, L = 2^b - 1, mean over every window lying
// inside the first valid_height rows).
//
// One CTA per 32x16 tile of window positions: the 42x26 pixel patch of both
// images goes to shared memory, a horizontal 11-tap pass forms the five local
// sums (x, y, x², y², xy) in float64 for 26 rows x 32 columns, the vertical
// pass finishes them per window and evaluates
//     ((2μxμy + C1)(2σxy + C2)) / ((μx² + μy² + C1)(σx² + σy² + C2)).
// Float64 keeps the variances (E[x²] − μ² of values up to 1023²) exact to
// ~1e-12.  The tile sum enters the per-image total as a 2^-32 fixed-point
// integer through a 64-bit atomic, so the result does not depend on the order
// in which tiles finish; a finaliser divides by the window count.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "internal.h"

namespace dct16a {
namespace {

constexpr int kSTW = 32, kSTH = 16;        // window positions per tile (columns, rows)
constexpr int kSPW = kSTW + 10, kSPH = kSTH + 10;   // pixels per patch
constexpr double kFix = 4294967296.0;      // 2^32

struct SsimParams {
    int W, VH, OW, OH, tiles_x, elem, N;
    long long pitch, istride;
    double g[11];   // normalised 1-D Gaussian, the 2-D window is g ⊗ g
    double C1, C2;
};

__device__ __forceinline__ float pix_at(const uint8_t* base, const SsimParams& p, int r, int c) {
    const uint8_t* row = base + r * p.pitch;
    return p.elem == 1 ? static_cast<float>(row[c]) : static_cast<float>(reinterpret_cast<const int16_t*>(row)[c]);
}

}  // namespace

__global__ void __launch_bounds__(256) ssim_kernel(const uint8_t* __restrict__ ref, const uint8_t* __restrict__ test,
                                                   unsigned long long* acc, const SsimParams p) {
    __shared__ float xs[kSPH][kSPW + 1], ys[kSPH][kSPW + 1];
    __shared__ double hs[5][kSPH][kSTW + 1];
    __shared__ double red[8];
    const int ty = blockIdx.x / p.tiles_x, tx = blockIdx.x - ty * p.tiles_x;
    for (int n = blockIdx.y; n < p.N; n += gridDim.y) {
    const int r0 = ty * kSTH, c0 = tx * kSTW;
    const uint8_t* a = ref + n * p.istride;
    const uint8_t* b = test + n * p.istride;
    for (int i = threadIdx.x; i < kSPH * kSPW; i += blockDim.x) {
        const int r = i / kSPW, c = i - r * kSPW;
        const int gr = r0 + r, gc = c0 + c;
        const bool in = gr < p.VH && gc < p.W;
        xs[r][c] = in ? pix_at(a, p, gr, gc) : 0.0f;
        ys[r][c] = in ? pix_at(b, p, gr, gc) : 0.0f;
    }
    __syncthreads();
    // horizontal pass: 26 rows x 32 window columns, five sums each
    for (int i = threadIdx.x; i < kSPH * kSTW; i += blockDim.x) {
        const int r = i / kSTW, c = i - r * kSTW;
        double sx = 0, sy = 0, sxx = 0, syy = 0, sxy = 0;
#pragma unroll
        for (int v = 0; v < 11; ++v) {
            const double x = xs[r][c + v], y = ys[r][c + v], w = p.g[v];
            sx = fma(w, x, sx);
            sy = fma(w, y, sy);
            sxx = fma(w, x * x, sxx);
            syy = fma(w, y * y, syy);
            sxy = fma(w, x * y, sxy);
        }
        hs[0][r][c] = sx;
        hs[1][r][c] = sy;
        hs[2][r][c] = sxx;
        hs[3][r][c] = syy;
        hs[4][r][c] = sxy;
    }
    __syncthreads();
    // vertical pass and the SSIM of each window
    double sum = 0.0;
    for (int i = threadIdx.x; i < kSTH * kSTW; i += blockDim.x) {
        const int r = i / kSTW, c = i - r * kSTW;
        if (r0 + r >= p.OH || c0 + c >= p.OW) continue;
        double m[5] = {0, 0, 0, 0, 0};
#pragma unroll
        for (int u = 0; u < 11; ++u) {
#pragma unroll
            for (int q = 0; q < 5; ++q) m[q] = fma(p.g[u], hs[q][r + u][c], m[q]);
        }
        const double mx = m[0], my = m[1];
        const double vx = m[2] - mx * mx, vy = m[3] - my * my, cxy = m[4] - mx * my;
        sum += ((2.0 * mx * my + p.C1) * (2.0 * cxy + p.C2)) / ((mx * mx + my * my + p.C1) * (vx + vy + p.C2));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sum;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) s += red[w];
        atomicAdd(acc + n, static_cast<unsigned long long>(llrint(s * kFix)));
    }
    __syncthreads();   // the patch and red[] are reused by the next image
    }
}

__global__ void ssim_finish_kernel(double* out, int n, double count) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const long long v = static_cast<long long>(reinterpret_cast<unsigned long long*>(out)[i]);
    out[i] = static_cast<double>(v) / kFix / count;
}

int launch_ssim(const void* ref, const void* test, const Geom& g, double* ssim, cudaStream_t st) {
    SsimParams p{};
    p.W = g.W;
    p.VH = g.VH;
    p.OW = g.W - 10;
    p.OH = g.VH - 10;
    p.tiles_x = (p.OW + kSTW - 1) / kSTW;
    p.elem = g.elem;
    p.N = g.N;
    p.pitch = g.pitch;
    p.istride = g.istride;
    double s = 0.0;
    for (int v = 0; v < 11; ++v) {
        p.g[v] = exp(-((v - 5) * (v - 5)) / (2.0 * 1.5 * 1.5));
        s += p.g[v];
    }
    for (int v = 0; v < 11; ++v) p.g[v] /= s;
    const double L = static_cast<double>((1 << g.bits) - 1);
    p.C1 = (0.01 * L) * (0.01 * L);
    p.C2 = (0.03 * L) * (0.03 * L);
    cudaError_t e = cudaMemsetAsync(ssim, 0, sizeof(double) * g.N, st);
    if (e) return static_cast<int>(e);
    const int tiles = p.tiles_x * ((p.OH + kSTH - 1) / kSTH);
    ssim_kernel<<<dim3(tiles, g.N < 65535 ? g.N : 65535), 256, 0, st>>>(static_cast<const uint8_t*>(ref), static_cast<const uint8_t*>(test),
                                                reinterpret_cast<unsigned long long*>(ssim), p);
    e = cudaGetLastError();
    if (e) return static_cast<int>(e);
    ssim_finish_kernel<<<(g.N + 127) / 128, 128, 0, st>>>(ssim, g.N, static_cast<double>(p.OW) * p.OH);
    return static_cast<int>(cudaGetLastError());
}

}  // namespace dct16a
