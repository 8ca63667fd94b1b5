// tables.cuh — the constant tables of the quantisation stage, restated from the
// paper (no code shared with the CPU oracle):
//   g_k = (T·Tᵀ)_kk, the squares of the denominators of S = diag(1/sqrt(g_k))
//         printed at PAPER.md:315-329;
//   W_kl = 2304 / (g_k·g_l) — the exact integer weights of the zonal inverse
//         (S² = diag(1/g) absorbed into quantisation);
//   zig-zag rank of (k, l) — JPEG boustrophedon over anti-diagonals, reading A4
//         (PAPER.md:882-894 does not print the order).
#pragma once
#include <stdint.h>

namespace dct16a {

__host__ __device__ constexpr int g_of(int k) {
    // 1/S_kk² from PAPER.md:315-329: 1/4 -> 16, 1/sqrt(12) -> 12, 1/sqrt(8) -> 8
    return k == 0 || k == 1 || k == 5 || k == 8 ? 16
         : (k == 3 || k == 4 || k == 11 || k == 12) ? 8
                                                    : 12;
}

// rank of (k, l) in the 16x16 zig-zag scan (0 = DC, 255 = (15,15))
__host__ __device__ constexpr int zigzag_rank(int k, int l) {
    const int d = k + l;
    const int before = d <= 15 ? d * (d + 1) / 2 : 256 - (31 - d) * (32 - d) / 2;
    const int kmin = d > 15 ? d - 15 : 0;
    const int kmax = d < 15 ? d : 15;
    // odd diagonals run with the row index increasing, even ones decreasing
    return before + ((d & 1) ? (k - kmin) : (kmax - k));
}

__host__ __device__ constexpr int w_of(int k, int l) { return 2304 / (g_of(k) * g_of(l)); }

}  // namespace dct16a
