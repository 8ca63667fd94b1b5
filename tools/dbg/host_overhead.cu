// host_overhead.cu — host-side cost of one C-ABI call (no Python): config-1
// sized work (one 512x512 u8 image), back-to-back calls on one stream, wall
// time per call (the GPU work of each call is a few µs, so the loop measures
// the host path once the queue is full), plus one call + sync latency.
// Build: nvcc -O2 -std=c++17 -I include tools/dbg/host_overhead.cu -o build/host_overhead
//        -Lpaper_1606_05562_b200 -ldct16a -Xlinker -rpath=$PWD/paper_1606_05562_b200
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <chrono>
#include <vector>

#include <cuda.h>

#include "dct16a.h"

__global__ void empty_kernel(int* p) {
    if (p) *p = 0;
}

template <class F>
double per_call_us(F f, int n) {
    for (int i = 0; i < 50; ++i) f();
    cudaDeviceSynchronize();
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < n; ++i) f();
    cudaDeviceSynchronize();
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count() / n;
}

int main() {
    const int W = 512, H = 512;
    std::vector<uint8_t> h(W * H);
    for (int i = 0; i < W * H; ++i) h[i] = uint8_t((i * 2654435761u) >> 24);
    uint8_t *src, *rec;
    int32_t* coef;
    uint64_t* sse;
    double* psnr;
    cudaMalloc(&src, W * H);
    cudaMalloc(&rec, W * H);
    cudaMalloc(&coef, W * H * 4);
    cudaMalloc(&sse, 8);
    cudaMalloc(&psnr, 8);
    cudaMemcpy(src, h.data(), W * H, cudaMemcpyHostToDevice);
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    dct16a_desc d = {W, H, H, 1, 8, 0, W, int64_t(W) * H};
    dct16a_quant q = {DCT16A_ZONAL, 16, 16, 0};
    printf("dct16a_codec (recon, sse, psnr): %.2f us/call\n",
           per_call_us([&] { dct16a_codec(src, &d, &q, rec, sse, psnr, st); }, 20000));
    printf("dct16a_codec (sse only):         %.2f us/call\n",
           per_call_us([&] { dct16a_codec(src, &d, &q, nullptr, sse, nullptr, st); }, 20000));
    printf("dct16a_forward:                  %.2f us/call\n",
           per_call_us([&] { dct16a_forward(src, &d, coef, st); }, 20000));
    printf("validation only (bad quant r=0): %.2f us/call\n", per_call_us([&] {
               dct16a_quant b = q;
               b.r = 0;
               dct16a_codec(src, &d, &b, rec, sse, psnr, st);
           }, 20000));
    printf("cudaMemsetAsync 8 B:             %.2f us/call\n",
           per_call_us([&] { cudaMemsetAsync(sse, 0, 8, st); }, 20000));
    {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult qr;
        cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr);
        using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                      const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
        EncodeFn enc = reinterpret_cast<EncodeFn>(fn);
        CUtensorMap m;
        cuuint64_t dims[3] = {cuuint64_t(W), cuuint64_t(H), 1}, str[2] = {cuuint64_t(W), cuuint64_t(W) * H};
        cuuint32_t box[3] = {128, 16, 1}, es[3] = {1, 1, 1};
        printf("cuTensorMapEncodeTiled:          %.2f us/call\n", per_call_us([&] {
                   enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, src, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
               }, 20000));
        cudaEvent_t ev;
        cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
        printf("cudaEventRecord:                 %.2f us/call\n", per_call_us([&] { cudaEventRecord(ev, st); }, 20000));
        cudaStreamCaptureStatus cs;
        printf("cudaStreamIsCapturing:           %.2f us/call\n", per_call_us([&] { cudaStreamIsCapturing(st, &cs); }, 20000));
        int dv;
        printf("cudaGetDevice:                   %.2f us/call\n", per_call_us([&] { cudaGetDevice(&dv); }, 20000));
        printf("empty kernel launch:             %.2f us/call\n", per_call_us([&] { empty_kernel<<<1, 32, 0, st>>>(nullptr); }, 20000));
        printf("empty launch, 8 KB of params:    (see codec)\n");
    }
    printf("call + stream sync:              %.2f us\n", per_call_us([&] {
               dct16a_codec(src, &d, &q, rec, sse, psnr, st);
               cudaStreamSynchronize(st);
           }, 2000));
    return 0;
}
