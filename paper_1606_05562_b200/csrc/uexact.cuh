// uexact.cuh — exact decisions of the uniform path (readings A6, A9, A10 of
// DESIGN.md §3), used only on the rare near-tie branch of the kernels.
//
// Reconstruction: with s_k = 1/sqrt(g_k) (S of PAPER.md:315-329) write
// 12·s_k = e_k·ρ_k, (e, ρ²) = (3, 1) for g = 16, (2, 3) for g = 12, (3, 2) for
// g = 8.  Then 144·s_k·s_l = e_k·e_l·ρ_k·ρ_l and
//     144·A′/Δ = J1 + J2·√2 + J3·√3 + J6·√6,
// J_d = Σ_kl T_ki·T_lj·q_kl·K_d(k, l) with integer K_d: equal classes give the
// rational cell e_k·e_l·ρ_k² (d = 1); classes (16,12), (16,8), (12,8) give
// ρ_kρ_l = √3, √2, √6 with K = e_k·e_l.  The sign of
//     144·(A′ + 1/2 − N)/Δ·Δ = b0 + b1·√2 + b2·√3 + b3·√6
// is decided in exact integer arithmetic (128-bit where squares need it):
// sign(P + Q·√3) with P = b0 + b1·√2, Q = b2 + b3·√2; opposite signs compare
// P² with 3Q² = R + S·√2.  Nothing here is shared with the CPU oracle, which
// decides the same pixels with square-free splits and 60-digit decimals.
#pragma once
#include <stdint.h>

#include "net16.cuh"
#include "quant.cuh"
#include "tables.cuh"

namespace dct16a {

__device__ __forceinline__ int uclass(int k) { return g_class(k); }   // 0, 1, 2 for g = 16, 12, 8

// sign(a + b·√2), exact
__device__ __forceinline__ int sign_r2(__int128 a, __int128 b) {
    if (a == 0 && b == 0) return 0;
    if (a >= 0 && b >= 0) return 1;
    if (a <= 0 && b <= 0) return -1;
    const unsigned __int128 ua = static_cast<unsigned __int128>(a < 0 ? -a : a);
    const unsigned __int128 ub = static_cast<unsigned __int128>(b < 0 ? -b : b);
    // |a|, |b| < 2^63 here, so the squares fit 128 bits
    return ua * ua > 2 * ub * ub ? (a > 0 ? 1 : -1) : (b > 0 ? 1 : -1);
}

// sign(b0 + b1·√2 + b2·√3 + b3·√6), exact; |b_i| < 2^30
__device__ __forceinline__ int sign_q23(long long b0, long long b1, long long b2, long long b3) {
    const int sp = sign_r2(b0, b1), sq = sign_r2(b2, b3);
    if (sq == 0) return sp;
    if (sp == 0 || sp == sq) return sq;
    const __int128 R = static_cast<__int128>(b0) * b0 + 2 * static_cast<__int128>(b1) * b1 -
                       3 * static_cast<__int128>(b2) * b2 - 6 * static_cast<__int128>(b3) * b3;
    const __int128 S = 2 * static_cast<__int128>(b0) * b1 - 6 * static_cast<__int128>(b2) * b3;
    return sign_r2(R, S) > 0 ? sp : sq;
}

// T as a table, built at compile time: column i of T = net_fwd(e_i) (the
// network of Eq. (1)).
struct TTable {
    int8_t v[16][16];
};
constexpr TTable make_t_table() {
    TTable t{};
    for (int i = 0; i < 16; ++i) {
        int32_t x[16] = {}, y[16] = {};
        x[i] = 1;
        net_fwd(x, y);
        for (int k = 0; k < 16; ++k) t.v[k][i] = static_cast<int8_t>(y[k]);
    }
    return t;
}
static __constant__ TTable c_T = make_t_table();

// floor(A′[i][j] + 1/2) exactly, for the levels q (q[k·qs + l], row stride qs)
// and step Δ, given N0 = the integer nearest to the float64 value of A′ + 1/2.
static __device__ __noinline__ int uniform_exact_floor(const int32_t* q, int i, int j, int step, int N0, int qs = 16) {
    const auto& T = c_T.v;
    const int e[3] = {3, 2, 3};
    const int r2[3] = {1, 3, 2};
    long long J1 = 0, J2 = 0, J3 = 0, J6 = 0;
    for (int k = 0; k < 16; ++k) {
        if (T[k][i] == 0) continue;
        const int ck = uclass(k);
        for (int l = 0; l < 16; ++l) {
            const int v = q[k * qs + l];
            if (v == 0 || T[l][j] == 0) continue;
            const int cl = uclass(l);
            const long long t = static_cast<long long>(T[k][i] * T[l][j]) * v * (e[ck] * e[cl]);
            if (ck == cl) J1 += t * r2[ck];
            else if (ck + cl == 1) J3 += t;      // classes (16, 12): √3
            else if (ck + cl == 2) J2 += t;      // (16, 8): √2
            else J6 += t;                        // (12, 8): √6
        }
    }
    const long long b0 = step * J1 + 72 - 144LL * N0;
    return sign_q23(b0, step * J2, step * J3, step * J6) >= 0 ? N0 : N0 - 1;
}

// floor(A′ + 1/2) exactly when every nonzero level of the block lies in a
// rational cell (g_k = g_l): then A′ = Δ·J1/144 with J1 an integer (the √2, √3,
// √6 components vanish), recovered from the float64 value a of A′ (|error| far
// below 1/2 unit of J1), and floor((Δ·J1 + 72)/144) is integer arithmetic.
__device__ __forceinline__ int uniform_rational_floor(double a, int step) {
    const long long J1 = __double2ll_rn(a * 144.0 / step);
    const long long num = static_cast<long long>(step) * J1 + 72;
    return static_cast<int>(num >= 0 ? num / 144 : -((-num + 143) / 144));
}

// Rounding of a float64 reconstruction value a = A′ (reading A6): floor(a + 1/2)
// through one round-down add onto 1.5·2^20 + 1/2 (ulp 2^-32): the high word
// carries 2^19 + floor(a + 1/2), the low word the 32 fraction bits.  `near` is
// set when the fraction lies within 2^-20 of an integer (float64 error of the
// butterfly evaluation is below 1e-9), where the caller decides exactly.
// Valid for |a| < 2^19.
__device__ __forceinline__ int round_f64(double a, bool& near, int& N0) {
    const double d = __dadd_rd(a, 1572864.5);
    const int hi = __double2hiint(d);
    const uint32_t lo = static_cast<uint32_t>(__double2loint(d));
    const int p = hi - 0x41380000;
    near = (lo + 4096u) < 8192u;
    N0 = p + (lo >> 31);
    return p;
}

}  // namespace dct16a
