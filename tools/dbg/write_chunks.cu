#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr long long N4 = 4096LL * 512 * 512 / 4;   // int4 elements of 4 GiB
// torch-like: CTA b writes int4 [b*per, (b+1)*per), thread t elements t + k*blockDim
template <int PER_THREAD>
__global__ void chunk_w(int4* __restrict__ out, long long n) {
    const long long base = (long long)blockIdx.x * blockDim.x * PER_THREAD;
#pragma unroll
    for (int k = 0; k < PER_THREAD; ++k) {
        long long i = base + threadIdx.x + (long long)k * blockDim.x;
        if (i < n) out[i] = make_int4((int)i, 1, 2, 3);
    }
}
// mix: CTA reads its u8 chunk (as uint32 words) and writes the int32 expansion
template <int PER_THREAD>
__global__ void chunk_mix(const uint32_t* __restrict__ in, int4* __restrict__ out, long long n4) {
    const long long base = (long long)blockIdx.x * blockDim.x * PER_THREAD;
    uint32_t v[PER_THREAD];
#pragma unroll
    for (int k = 0; k < PER_THREAD; ++k) {
        long long i = base + threadIdx.x + (long long)k * blockDim.x;
        v[k] = i < n4 ? __ldcs(in + i) : 0;
    }
#pragma unroll
    for (int k = 0; k < PER_THREAD; ++k) {
        long long i = base + threadIdx.x + (long long)k * blockDim.x;
        if (i < n4) out[i] = make_int4(v[k] & 255, (v[k] >> 8) & 255, (v[k] >> 16) & 255, v[k] >> 24);
    }
}
template <class F> float timeit(F f) {
    f(); cudaDeviceSynchronize(); cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a); for (int r = 0; r < 20; ++r) f(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); return ms / 20;
}
int main() {
    int4* out; uint32_t* in; cudaMalloc(&out, N4 * 16); cudaMalloc(&in, N4 * 4); cudaMemset(in, 3, N4 * 4);
    for (int tpb : {128, 256, 512}) {
        auto run = [&](auto kern, int per) { long long g = (N4 + (long long)tpb * per - 1) / ((long long)tpb * per);
            return timeit([&]{ kern<<<(unsigned)g, tpb>>>(out, N4); }); };
        printf("write chunk tpb %d per 1: %.1f GB/s\n", tpb, N4 * 16.0 / run(chunk_w<1>, 1) / 1e6);
        printf("write chunk tpb %d per 4: %.1f GB/s\n", tpb, N4 * 16.0 / run(chunk_w<4>, 4) / 1e6);
        printf("write chunk tpb %d per 16: %.1f GB/s\n", tpb, N4 * 16.0 / run(chunk_w<16>, 16) / 1e6);
        auto runm = [&](auto kern, int per) { long long g = (N4 + (long long)tpb * per - 1) / ((long long)tpb * per);
            return timeit([&]{ kern<<<(unsigned)g, tpb>>>(in, out, N4); }); };
        printf("mix chunk tpb %d per 1: %.1f GB/s\n", tpb, N4 * 20.0 / runm(chunk_mix<1>, 1) / 1e6);
        printf("mix chunk tpb %d per 4: %.1f GB/s\n", tpb, N4 * 20.0 / runm(chunk_mix<4>, 4) / 1e6);
        printf("mix chunk tpb %d per 8: %.1f GB/s\n", tpb, N4 * 20.0 / runm(chunk_mix<8>, 8) / 1e6);
        printf("mix chunk tpb %d per 16: %.1f GB/s\n", tpb, N4 * 20.0 / runm(chunk_mix<16>, 16) / 1e6);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
