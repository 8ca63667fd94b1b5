// mc_single.cu — the NVLS multicast form of the fused SSE all-reduce executed
// on ONE GPU: a one-device multicast object (driver API, one process, no
// handle export) is bound to device memory, the codec kernel adds every
// frame's SSE with multimem.red through the multicast address
// (dct16a_codec_allreduce_multicast), and the unicast view must equal the SSE
// that dct16a_codec computes (itself oracle-checked by the GPU tests).
// Build: nvcc -O2 -std=c++17 -I include tools/dbg/mc_single.cu -o build/mc_single
//        -Lpaper_1606_05562_b200 -ldct16a -lcuda -Xlinker -rpath=$PWD/paper_1606_05562_b200
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>

#include "dct16a.h"

#define CK(x)                                                                         \
    do {                                                                              \
        CUresult r_ = (x);                                                            \
        if (r_ != CUDA_SUCCESS) {                                                     \
            const char* s_ = nullptr;                                                 \
            cuGetErrorString(r_, &s_);                                                \
            printf("FAIL %s -> %d %s\n", #x, int(r_), s_ ? s_ : "?");                 \
            return 3;                                                                 \
        }                                                                             \
    } while (0)
#define RK(x)                                                                         \
    do {                                                                              \
        cudaError_t r_ = (x);                                                         \
        if (r_ != cudaSuccess) {                                                      \
            printf("FAIL %s -> %s\n", #x, cudaGetErrorString(r_));                    \
            return 3;                                                                 \
        }                                                                             \
    } while (0)
#define LK(x)                                                                         \
    do {                                                                              \
        int r_ = (x);                                                                 \
        if (r_ != 0) {                                                                \
            printf("FAIL %s -> %d %s\n", #x, r_, dct16a_last_error());                \
            return 3;                                                                 \
        }                                                                             \
    } while (0)

int main() {
    RK(cudaSetDevice(0));
    RK(cudaFree(0));   // primary context
    CUdevice dev;
    CK(cuDeviceGet(&dev, 0));
    int mc_ok = 0;
    CK(cuDeviceGetAttribute(&mc_ok, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
    if (!mc_ok) {
        printf("SKIP multicast not supported\n");
        return 2;
    }
    CUmulticastObjectProp mp = {};
    mp.numDevices = 1;
    mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;   // required field; never exported
    size_t gran = 0;
    CK(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
    const size_t size = gran;   // one granule holds the SSE vector
    mp.size = size;
    CUmemGenericAllocationHandle mc, mem;
    CK(cuMulticastCreate(&mc, &mp));
    CK(cuMulticastAddDevice(mc, dev));
    CUmemAllocationProp ap = {};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = 0;
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    CK(cuMemCreate(&mem, size, &ap, 0));
    CK(cuMulticastBindMem(mc, 0, mem, 0, size, 0));
    CUmemAccessDesc acc = {};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = 0;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CUdeviceptr uc = 0, mcp = 0;
    CK(cuMemAddressReserve(&uc, size, gran, 0, 0));
    CK(cuMemMap(uc, size, 0, mem, 0));
    CK(cuMemSetAccess(uc, size, &acc, 1));
    CK(cuMemAddressReserve(&mcp, size, gran, 0, 0));
    CK(cuMemMap(mcp, size, 0, mc, 0));
    CK(cuMemSetAccess(mcp, size, &acc, 1));

    // 12 frames of 256 x 384 10-bit pixels: a smooth field plus a hashed texture
    const int n = 12, H = 256, W = 384;
    std::vector<int16_t> h(size_t(n) * H * W);
    for (int f = 0; f < n; ++f)
        for (int y = 0; y < H; ++y)
            for (int x = 0; x < W; ++x) {
                uint32_t k = uint32_t(f * 2654435761u) ^ uint32_t(y * 40503u) ^ uint32_t(x * 9973u);
                k ^= k >> 13;
                k *= 0x5bd1e995u;
                k ^= k >> 15;
                const int v = 512 + int(300.0 * ((x + 2 * y + 37 * f) % 97) / 97.0) - 150 + int(k % 61) - 30;
                h[(size_t(f) * H + y) * W + x] = int16_t(v < 0 ? 0 : (v > 1023 ? 1023 : v));
            }
    int16_t* d_src = nullptr;
    uint64_t* d_sse = nullptr;
    RK(cudaMalloc(&d_src, h.size() * 2));
    RK(cudaMalloc(&d_sse, n * 8));
    RK(cudaMemcpy(d_src, h.data(), h.size() * 2, cudaMemcpyHostToDevice));
    dct16a_desc d = {W, H, H, n, 10, 0, int64_t(W) * 2, int64_t(W) * H * 2};
    dct16a_quant q = {DCT16A_UNIFORM, 16, 16, 0};
    CK(cuMemsetD8(uc, 0, size));
    const int64_t off = 5;
    LK(dct16a_codec_allreduce_multicast(d_src, &d, &q, nullptr, reinterpret_cast<uint64_t*>(mcp), off, nullptr));
    LK(dct16a_codec(d_src, &d, &q, nullptr, d_sse, nullptr, nullptr));
    RK(cudaDeviceSynchronize());
    std::vector<uint64_t> got(64), ref(n);
    CK(cuMemcpyDtoH(got.data(), uc, 64 * 8));
    RK(cudaMemcpy(ref.data(), d_sse, n * 8, cudaMemcpyDeviceToHost));
    bool ok = true;
    for (int i = 0; i < 64; ++i) ok &= got[i] == (i >= off && i < off + n ? ref[i - off] : 0);
    // two more runs: multimem.red adds onto the vector
    LK(dct16a_codec_allreduce_multicast(d_src, &d, &q, nullptr, reinterpret_cast<uint64_t*>(mcp), off, nullptr));
    LK(dct16a_codec_allreduce_multicast(d_src, &d, &q, nullptr, reinterpret_cast<uint64_t*>(mcp), off, nullptr));
    RK(cudaDeviceSynchronize());
    CK(cuMemcpyDtoH(got.data(), uc, 64 * 8));
    bool ok3 = true;
    for (int i = 0; i < n; ++i) ok3 &= got[off + i] == 3 * ref[i];
    printf("multicast (1-device NVLS object, granule %zu B): SSE via multimem.red %s; x3 after three runs %s; "
           "frame 0 SSE %llu\n",
           gran, ok ? "EQUAL" : "DIFFERENT", ok3 ? "EQUAL" : "DIFFERENT", (unsigned long long)ref[0]);
    return ok && ok3 ? 0 : 1;
}
