/*
 * c_api_demo.c — the C ABI of include/dct16a.h used from plain C (no Python,
 * no torch): forward transform, fused zonal codec, PSNR and SSIM on a small
 * synthetic batch, with checks that need no oracle:
 *   - Z_00 of every block equals the block sum (row 0 of T is all ones,
 *     PAPER.md:272);
 *   - integer Parseval: sum W_kl·Z_kl² = 2304·sum X² with W = 2304/(g_k g_l)
 *     (T·Tᵀ = diag(g));
 *   - the SSE reported by dct16a_codec equals dct16a_psnr on its output;
 *   - r = 256 reconstructs the input exactly (SSE 0, PSNR +inf, SSIM 1).
 * Build: gcc -O2 -I include examples/c_api_demo.c -L paper_1606_05562_b200 -ldct16a \
 *            -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,<those dirs> -o c_api_demo
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime_api.h>

#include "dct16a.h"

#define CHECK(x)                                                                  \
    do {                                                                          \
        int rc_ = (x);                                                            \
        if (rc_) {                                                                \
            fprintf(stderr, "%s failed: %d %s\n", #x, rc_, dct16a_last_error()); \
            return 1;                                                             \
        }                                                                         \
    } while (0)
#define CUDA(x)                                                                        \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess) {                                                       \
            fprintf(stderr, "%s failed: %s\n", #x, cudaGetErrorString(e_));            \
            return 1;                                                                  \
        }                                                                              \
    } while (0)

static int g_of(int k) {   /* diag(T·Tᵀ) */
    return (k == 0 || k == 1 || k == 5 || k == 8) ? 16 : ((k == 3 || k == 4 || k == 11 || k == 12) ? 8 : 12);
}

int main(void) {
    const int N = 3, H = 64, W = 96;
    const size_t npx = (size_t)N * H * W, nblk = (size_t)N * (H / 16) * (W / 16);
    uint8_t* img = (uint8_t*)malloc(npx);
    uint32_t s = 12345u;
    for (size_t i = 0; i < npx; ++i) {   /* smooth ramp plus LCG noise */
        s = s * 1664525u + 1013904223u;
        img[i] = (uint8_t)((i % W) + (i / W % H) + (s >> 28));
    }
    void *d_img, *d_rec;
    int32_t* d_coef;
    uint64_t* d_sse;
    double *d_psnr, *d_ssim;
    CUDA(cudaMalloc(&d_img, npx));
    CUDA(cudaMalloc(&d_rec, npx));
    CUDA(cudaMalloc((void**)&d_coef, nblk * 256 * sizeof(int32_t)));
    CUDA(cudaMalloc((void**)&d_sse, 2 * N * sizeof(uint64_t)));
    CUDA(cudaMalloc((void**)&d_psnr, N * sizeof(double)));
    CUDA(cudaMalloc((void**)&d_ssim, N * sizeof(double)));
    CUDA(cudaMemcpy(d_img, img, npx, cudaMemcpyHostToDevice));

    dct16a_desc d;
    memset(&d, 0, sizeof d);
    d.width = W;
    d.height = H;
    d.valid_height = H;
    d.batch = N;
    d.bit_depth = 8;
    d.pitch_bytes = W;
    d.image_stride_bytes = (int64_t)W * H;
    printf("%s\n", dct16a_version());

    /* forward: DC = block sum, integer Parseval */
    CHECK(dct16a_forward(d_img, &d, d_coef, NULL));
    int32_t* coef = (int32_t*)malloc(nblk * 256 * sizeof(int32_t));
    CUDA(cudaMemcpy(coef, d_coef, nblk * 256 * sizeof(int32_t), cudaMemcpyDeviceToHost));
    int bad = 0;
    for (size_t b = 0; b < nblk; ++b) {
        const int n = (int)(b / ((H / 16) * (W / 16))), rem = (int)(b % ((H / 16) * (W / 16)));
        const int by = rem / (W / 16), bx = rem % (W / 16);
        long long sum = 0, sq = 0, wz = 0;
        for (int i = 0; i < 16; ++i)
            for (int j = 0; j < 16; ++j) {
                const long long v = img[(size_t)n * W * H + (size_t)(by * 16 + i) * W + bx * 16 + j];
                sum += v;
                sq += v * v;
            }
        for (int k = 0; k < 16; ++k)
            for (int l = 0; l < 16; ++l) {
                const long long z = coef[b * 256 + 16 * k + l];
                wz += (2304 / (g_of(k) * g_of(l))) * z * z;
            }
        bad += coef[b * 256] != sum;
        bad += wz != 2304 * sq;
    }
    printf("forward: %zu blocks, DC/Parseval mismatches: %d\n", nblk, bad);

    /* fused codec vs psnr, SSIM; and r = 256 lossless */
    dct16a_quant q = {DCT16A_ZONAL, 16, 16, 0};
    CHECK(dct16a_codec(d_img, &d, &q, d_rec, d_sse, d_psnr, NULL));
    CHECK(dct16a_psnr(d_img, d_rec, &d, d_sse + N, NULL, NULL));
    CHECK(dct16a_ssim(d_img, d_rec, &d, d_ssim, NULL));
    uint64_t sse[6];
    double psnr[3], ssim[3];
    CUDA(cudaMemcpy(sse, d_sse, sizeof sse, cudaMemcpyDeviceToHost));
    CUDA(cudaMemcpy(psnr, d_psnr, sizeof psnr, cudaMemcpyDeviceToHost));
    CUDA(cudaMemcpy(ssim, d_ssim, sizeof ssim, cudaMemcpyDeviceToHost));
    for (int n = 0; n < N; ++n) {
        printf("r=16 image %d: SSE %llu (psnr kernel %llu)  PSNR %.4f dB  SSIM %.5f\n", n,
               (unsigned long long)sse[n], (unsigned long long)sse[N + n], psnr[n], ssim[n]);
        bad += sse[n] != sse[N + n];
    }
    q.r = 256;
    CHECK(dct16a_codec(d_img, &d, &q, d_rec, d_sse, d_psnr, NULL));
    CHECK(dct16a_ssim(d_img, d_rec, &d, d_ssim, NULL));
    CUDA(cudaMemcpy(sse, d_sse, N * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    CUDA(cudaMemcpy(psnr, d_psnr, sizeof psnr, cudaMemcpyDeviceToHost));
    CUDA(cudaMemcpy(ssim, d_ssim, sizeof ssim, cudaMemcpyDeviceToHost));
    for (int n = 0; n < N; ++n) bad += sse[n] != 0 || !isinf(psnr[n]) || ssim[n] != 1.0;
    printf("r=256: SSE %llu PSNR %f SSIM %f\n", (unsigned long long)sse[0], psnr[0], ssim[0]);

    /* a validation error: r = 0 is a domain error, nothing is launched */
    q.r = 0;
    const int rc = dct16a_codec(d_img, &d, &q, d_rec, d_sse, d_psnr, NULL);
    printf("r=0 -> %d (%s)\n", rc, dct16a_last_error());
    bad += rc != DCT16A_EDOMAIN;
    CUDA(cudaDeviceSynchronize());
    printf(bad ? "c_api_demo FAILED (%d)\n" : "c_api_demo ok\n", bad);
    return bad != 0;
}
