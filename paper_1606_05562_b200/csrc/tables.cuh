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

// 1/S_kk² from PAPER.md:315-329: 1/4 -> 16 (k = 0, 1, 5, 8), 1/sqrt(12) -> 12,
// 1/sqrt(8) -> 8 (k = 3, 4, 11, 12), as the class c_k = (16 - g_k)/4 in two bits
// per k (branch-free for a runtime k: one shift, one mask)
constexpr uint32_t kGClassBits = 0x56945290u;
__host__ __device__ constexpr int g_class(int k) { return static_cast<int>((kGClassBits >> (2 * k)) & 3u); }
__host__ __device__ constexpr int g_of(int k) { return 16 - 4 * g_class(k); }
static_assert(g_of(0) == 16 && g_of(1) == 16 && g_of(5) == 16 && g_of(8) == 16 && g_of(3) == 8 &&
                  g_of(4) == 8 && g_of(11) == 8 && g_of(12) == 8 && g_of(2) == 12 && g_of(15) == 12,
              "g_k of PAPER.md:315-329");

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
