// quant.cuh — the quantisation stage with S folded in and
// the exact reconstruction decisions, shared by the standalone K4/K5 kernels
// and the fused codec (K2/K3).
//
//   s_k = 1/sqrt(g_k), g = diag(T·Tᵀ)             (S of PAPER.md:315-329)
//   zonal:   W_kl = 2304/(g_k·g_l) ∈ {9,12,16,18,24,36}, N = Tᵀ·(W ⊙ Z ⊙ M_r)·T,
//            pixel = clamp(round_half_away(N/2304))  (exact integers, reading A6)
//   uniform: q = sign(Z)·floor(|Z|/(Δ·sqrt(G)) + 1/2), G = g_k·g_l, decided
//            exactly (reading A9); B̂ = Δ·q·s_k·s_l; A′ = Tᵀ·B̂·T in float64 (A10)
#pragma once
#include <math.h>
#include <stdint.h>

#include "tables.cuh"

namespace dct16a {

// s_k as correctly rounded double literals: 1/4, 1/sqrt(12), 1/sqrt(8)
__host__ __device__ __forceinline__ double s_of(int k) {
    const int g = g_of(k);
    return g == 16 ? 0.25 : (g == 12 ? 0.2886751345948128822545743902509787 : 0.3535533905932737622004221810524245);
}

// Exact check of a uniform level candidate m >= 0 for |Z| = az:
// m is right iff (2m-1)²·Δ²·G <= 4·Z²  (m >= 1)  and  4·Z² < (2m+1)²·Δ²·G.
__device__ __forceinline__ int32_t uniform_fix(uint32_t az, int32_t m, uint64_t d2g) {
    const uint64_t z4 = 4ull * az * az;
    if (m > 0 && static_cast<uint64_t>(2 * m - 1) * static_cast<uint64_t>(2 * m - 1) * d2g > z4) return m - 1;
    if (static_cast<uint64_t>(2 * m + 1) * static_cast<uint64_t>(2 * m + 1) * d2g <= z4) return m + 1;
    return m;
}

// Uniform level m = floor(|Z|·c + 1/2) with c = 1/(Δ·sqrt(G)) in float: the
// float estimate is exact unless e lies within `margin` of an integer (exact ties
// of the rational cells land there too); those take the exact integer check.
// |e error| <= e·2^-22 < margin = 2^-11 + e·2^-20 guarantees at most one step off.
__device__ __forceinline__ int32_t uniform_level(int32_t z, float c, uint64_t d2g) {
    const uint32_t az = static_cast<uint32_t>(z < 0 ? -z : z);
    const float e = fmaf(static_cast<float>(az), c, 0.5f);
    const float fl = floorf(e);
    int32_t m = static_cast<int32_t>(fl);
    const float fr = e - fl;
    const float margin = 4.8828125e-4f + e * 9.5367431640625e-7f;
    if (fr < margin || fr > 1.0f - margin) m = uniform_fix(az, m, d2g);
    return z < 0 ? -m : m;
}

// cvt.pack.sat: (sat_u8(a) << 8) | sat_u8(b) | (c << 16); saturation clamps to [0, 255]
__device__ __forceinline__ uint32_t pack2_sat_u8(int a, int b, uint32_t c) {
    uint32_t d;
    asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

__device__ __forceinline__ int zonal_pixel(int32_t N, int maxpix) {
    // round half away of N/2304, clamped to [0, maxpix] (reading A6)
    const int32_t v = N + 1152;
    if (v <= 0) return 0;
    const int32_t p = static_cast<int32_t>(static_cast<uint32_t>(v) / 2304u);
    return p > maxpix ? maxpix : p;
}


}  // namespace dct16a
