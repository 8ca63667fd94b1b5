// net16.cuh — the 16-point butterfly networks of arXiv 1606.05562, Eq. (1)
// (PAPER.md:347-469): y = T·x = P2·M4·M3·M2·P1·M1·x with 60 additions and no
// multiplications (Table 1), and its transpose x = Tᵀ·y (also 60
// additions).  The networks are written once, generic over the value type:
//   * uint32_t carrying two 16-bit lanes (SWAR): lo + hi·2^16 is linear under
//     +/-, so one network evaluates two independent vectors (mod 2^32 wrap is
//     intended and well defined for unsigned arithmetic);
//   * int32_t, float (exact below 2^24), double.
#pragma once
#include <stdint.h>

namespace dct16a {

// Forward network, stage by stage as printed in Eq. (1).
template <typename V>
__device__ __forceinline__ void net_fwd(const V (&x)[16], V (&y)[16]) {
    // M1 = [[I8, Ī8], [Ī8, -I8]]: 16 additions
    const V a0 = x[0] + x[15], a1 = x[1] + x[14], a2 = x[2] + x[13], a3 = x[3] + x[12];
    const V a4 = x[4] + x[11], a5 = x[5] + x[10], a6 = x[6] + x[9], a7 = x[7] + x[8];
    const V a8 = x[7] - x[8], a9 = x[6] - x[9], a10 = x[5] - x[10], a11 = x[4] - x[11];
    const V a12 = x[3] - x[12], a13 = x[2] - x[13], a14 = x[1] - x[14], a15 = x[0] - x[15];
    // P1 = diag(I9, 7x7 permutation): wiring only
    const V b0 = a0, b1 = a1, b2 = a2, b3 = a3, b4 = a4, b5 = a5, b6 = a6, b7 = a7, b8 = a8;
    const V b9 = a11, b10 = a12, b11 = a15, b12 = a14, b13 = a13, b14 = a10, b15 = a9;
    // M2 = diag(B8, B8), B8 = [[I4, Ī4], [Ī4, -I4]]: 16 additions
    const V c0 = b0 + b7, c1 = b1 + b6, c2 = b2 + b5, c3 = b3 + b4;
    const V c4 = b3 - b4, c5 = b2 - b5, c6 = b1 - b6, c7 = b0 - b7;
    const V c8 = b8 + b15, c9 = b9 + b14, c10 = b10 + b13, c11 = b11 + b12;
    const V c12 = b11 - b12, c13 = b10 - b13, c14 = b9 - b14, c15 = b8 - b15;
    // M3 = diag of four 4x4 blocks: 24 additions
    const V d0 = c0 + c3, d1 = c1 + c2, d2 = c2 - c1, d3 = c0 - c3;
    const V d4 = c5 + c6 + c7, d5 = c7 - c4 - c5, d6 = c5 - c4 - c6, d7 = c4 - c6 + c7;
    const V d8 = c8 + c11, d9 = c9 + c10, d10 = c10 - c9, d11 = c11 - c8;
    const V d12 = c13 + c14 + c15, d13 = c12 + c13 - c15, d14 = c12 - c13 + c14,
            d15 = c12 - c14 + c15;
    // M4 = diag(H2, I6, H2, I6): 4 additions
    const V e0 = d0 + d1, e1 = d0 - d1, e8 = d8 + d9, e9 = d8 - d9;
    // P2: y_i = e_sigma(i), sigma = (0)(1 8)(2 4 3 11 10 7 12)(5 9 13 14 6)(15)
    // (closure reading A1)
    y[0] = e0;  y[1] = e8;  y[2] = d4;  y[3] = d11; y[4] = d3;  y[5] = e9;  y[6] = d5;  y[7] = d12;
    y[8] = e1;  y[9] = d13; y[10] = d7; y[11] = d10; y[12] = d2; y[13] = d14; y[14] = d6; y[15] = d15;
}

// Transposed network x = Tᵀ·y = M1ᵀ·P1ᵀ·M2ᵀ·M3ᵀ·M4ᵀ·P2ᵀ·y (the signal-flow graph
// of Eq. (1) run backwards; M1, M2, M4 are symmetric).  60 additions.
template <typename V>
__device__ __forceinline__ void net_inv(const V (&y)[16], V (&x)[16]) {
    // P2ᵀ: u_sigma(i) = y_i
    const V u0 = y[0], u8 = y[1], u4 = y[2], u11 = y[3], u3 = y[4], u9 = y[5], u5 = y[6], u12 = y[7];
    const V u1 = y[8], u13 = y[9], u7 = y[10], u10 = y[11], u2 = y[12], u14 = y[13], u6 = y[14],
            u15 = y[15];
    // M4ᵀ = M4
    const V v0 = u0 + u1, v1 = u0 - u1, v8 = u8 + u9, v9 = u8 - u9;
    const V v2 = u2, v3 = u3, v4 = u4, v5 = u5, v6 = u6, v7 = u7;
    const V v10 = u10, v11 = u11, v12 = u12, v13 = u13, v14 = u14, v15 = u15;
    // M3ᵀ (blockwise transposes)
    const V w0 = v0 + v3, w1 = v1 - v2, w2 = v1 + v2, w3 = v0 - v3;
    const V w4 = v7 - v5 - v6, w5 = v4 - v5 + v6, w6 = v4 - v6 - v7, w7 = v4 + v5 + v7;
    const V w8 = v8 - v11, w9 = v9 - v10, w10 = v9 + v10, w11 = v8 + v11;
    const V w12 = v13 + v14 + v15, w13 = v12 + v13 - v14, w14 = v12 + v14 - v15,
            w15 = v12 - v13 + v15;
    // M2ᵀ = M2
    const V p0 = w0 + w7, p1 = w1 + w6, p2 = w2 + w5, p3 = w3 + w4;
    const V p4 = w3 - w4, p5 = w2 - w5, p6 = w1 - w6, p7 = w0 - w7;
    const V p8 = w8 + w15, p9 = w9 + w14, p10 = w10 + w13, p11 = w11 + w12;
    const V p12 = w11 - w12, p13 = w10 - w13, p14 = w9 - w14, p15 = w8 - w15;
    // P1ᵀ
    const V q0 = p0, q1 = p1, q2 = p2, q3 = p3, q4 = p4, q5 = p5, q6 = p6, q7 = p7, q8 = p8;
    const V q11 = p9, q12 = p10, q15 = p11, q14 = p12, q13 = p13, q10 = p14, q9 = p15;
    // M1ᵀ = M1
    x[0] = q0 + q15; x[1] = q1 + q14; x[2] = q2 + q13; x[3] = q3 + q12;
    x[4] = q4 + q11; x[5] = q5 + q10; x[6] = q6 + q9;  x[7] = q7 + q8;
    x[8] = q7 - q8;  x[9] = q6 - q9;  x[10] = q5 - q10; x[11] = q4 - q11;
    x[12] = q3 - q12; x[13] = q2 - q13; x[14] = q1 - q14; x[15] = q0 - q15;
}

}  // namespace dct16a
