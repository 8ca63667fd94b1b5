// mix_ceiling.cu — what HBM sustains for the byte mix of the config-2 forward
// (read 1 GiB of uint8, write 4 GiB of int32, 20/80) with no compute:
//   expand_lsu<U>:  grid-stride, each thread loads 4 px per step (LDG.32, a warp
//                   covers 128 contiguous bytes) and stores them as one 16-byte
//                   int4 (a warp covers 512 contiguous bytes), U steps unrolled;
//   expand_v4<U>:   each thread loads 16 px (LDG.128) and stores 4 x int4 at
//                   64-byte stride (a warp instruction covers 2 KB sparsely);
//   write_only / read_only / copy: the pure ceilings with the same LSU code.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mix_ceiling tools/mix_ceiling.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr long long kPix = 4096LL * 512 * 512;   // config 2

template <int U>
__global__ void expand_lsu(const uint32_t* __restrict__ in, int4* __restrict__ out, long long n4) {
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
    long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    for (; i + (U - 1) * stride < n4; i += U * stride) {
        uint32_t v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = __ldcs(in + i + u * stride);
#pragma unroll
        for (int u = 0; u < U; ++u)
            __stcs(out + i + u * stride, make_int4(v[u] & 255, (v[u] >> 8) & 255, (v[u] >> 16) & 255, v[u] >> 24));
    }
    for (; i < n4; i += stride) {
        const uint32_t v = __ldcs(in + i);
        __stcs(out + i, make_int4(v & 255, (v >> 8) & 255, (v >> 16) & 255, v >> 24));
    }
}

__global__ void expand_v4(const uint4* __restrict__ in, int4* __restrict__ out, long long n16) {
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n16; i += stride) {
        const uint4 v = __ldcs(in + i);
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int q = 0; q < 4; ++q)
            __stcs(out + 4 * i + q, make_int4(w[q] & 255, (w[q] >> 8) & 255, (w[q] >> 16) & 255, w[q] >> 24));
    }
}

__global__ void write_only(int4* __restrict__ out, long long n) {
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n; i += stride)
        __stcs(out + i, make_int4(static_cast<int>(i), 1, 2, 3));
}

__global__ void read_only(const int4* __restrict__ in, long long n, int* sink) {
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
    int acc = 0;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n; i += stride) {
        const int4 v = __ldcs(in + i);
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x12345678) *sink = acc;
}

template <class F>
float timeit(F f, int reps = 20) {
    f();
    cudaDeviceSynchronize();
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint8_t* in;
    int32_t* out;
    int* sink;
    cudaMalloc(&in, kPix);
    cudaMalloc(&out, kPix * 4);
    cudaMalloc(&sink, 4);
    cudaMemset(in, 7, kPix);
    const double mix = kPix * 5.0;
    for (int tpb : {256, 512, 1024})
        for (int bps : {1, 2, 4, 8}) {
            if (tpb * bps > 2048) continue;
            const int grid = sms * bps;
            float ms = timeit([&] { expand_lsu<4><<<grid, tpb>>>((const uint32_t*)in, (int4*)out, kPix / 4); });
            printf("expand_lsu<4> tpb %4d blocks/SM %d   %.3f ms  %.1f GB/s\n", tpb, bps, ms, mix / ms / 1e6);
        }
    for (int tpb : {256, 1024}) {
        const int grid = sms * (2048 / tpb);
        float ms = timeit([&] { expand_lsu<1><<<grid, tpb>>>((const uint32_t*)in, (int4*)out, kPix / 4); });
        printf("expand_lsu<1> tpb %4d full occ     %.3f ms  %.1f GB/s\n", tpb, ms, mix / ms / 1e6);
        ms = timeit([&] { expand_lsu<8><<<grid, tpb>>>((const uint32_t*)in, (int4*)out, kPix / 4); });
        printf("expand_lsu<8> tpb %4d full occ     %.3f ms  %.1f GB/s\n", tpb, ms, mix / ms / 1e6);
        ms = timeit([&] { expand_v4<<<grid, tpb>>>((const uint4*)in, (int4*)out, kPix / 16); });
        printf("expand_v4     tpb %4d full occ     %.3f ms  %.1f GB/s\n", tpb, ms, mix / ms / 1e6);
    }
    {
        const int grid = sms * 2;
        float ms = timeit([&] { write_only<<<grid, 1024>>>((int4*)out, kPix / 4); });
        printf("write_only 4 GiB                      %.3f ms  %.1f GB/s\n", ms, kPix * 4.0 / ms / 1e6);
        ms = timeit([&] { read_only<<<grid, 1024>>>((const int4*)out, kPix / 4, sink); });
        printf("read_only 4 GiB                       %.3f ms  %.1f GB/s\n", ms, kPix * 4.0 / ms / 1e6);
        ms = timeit([&] { cudaMemcpyAsync(out + kPix / 2, out, kPix * 2, cudaMemcpyDeviceToDevice); });
        printf("cudaMemcpy D2D 2 GiB                  %.3f ms  %.1f GB/s (r+w)\n", ms, kPix * 4.0 / ms / 1e6);
    }
    printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
