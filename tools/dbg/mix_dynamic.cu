#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr long long N4 = 4096LL * 512 * 512 / 4;
__device__ unsigned long long g_ctr;
template <int PER>
__device__ __forceinline__ void do_chunk(const uint32_t* __restrict__ in, int4* __restrict__ out, long long c, long long n4) {
    const long long base = c * blockDim.x * PER;
    uint32_t v[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) { long long i = base + threadIdx.x + (long long)k * blockDim.x; v[k] = i < n4 ? __ldcs(in + i) : 0; }
#pragma unroll
    for (int k = 0; k < PER; ++k) { long long i = base + threadIdx.x + (long long)k * blockDim.x;
        if (i < n4) out[i] = make_int4(v[k] & 255, (v[k] >> 8) & 255, (v[k] >> 16) & 255, v[k] >> 24); }
}
template <int PER>
__global__ void dyn(const uint32_t* __restrict__ in, int4* __restrict__ out, long long n4, long long nchunks) {
    __shared__ long long c;
    while (true) {
        if (threadIdx.x == 0) c = (long long)atomicAdd(&g_ctr, 1ULL);
        __syncthreads();
        long long my = c;
        __syncthreads();
        if (my >= nchunks) break;
        do_chunk<PER>(in, out, my, n4);
    }
}
template <int PER>
__global__ void stat(const uint32_t* __restrict__ in, int4* __restrict__ out, long long n4, long long nchunks) {
    for (long long c = blockIdx.x; c < nchunks; c += gridDim.x) do_chunk<PER>(in, out, c, n4);
}
template <class F> float timeit(F f) {
    f(); cudaDeviceSynchronize(); cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a); for (int r = 0; r < 20; ++r) f(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); return ms / 20;
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int4* out; uint32_t* in; cudaMalloc(&out, N4 * 16); cudaMalloc(&in, N4 * 4); cudaMemset(in, 3, N4 * 4);
    const int tpb = 256; const int PER = 4;
    long long nch = N4 / (tpb * PER);
    unsigned long long zero = 0;
    for (int bps : {2, 4, 8}) {
        int grid = sms * bps;
        float ms = timeit([&]{ cudaMemcpyToSymbolAsync(g_ctr, &zero, 8); dyn<PER><<<grid, tpb>>>(in, out, N4, nch); });
        printf("dynamic persistent blocks/SM %d: %.1f GB/s\n", bps, N4 * 20.0 / ms / 1e6);
        ms = timeit([&]{ stat<PER><<<grid, tpb>>>(in, out, N4, nch); });
        printf("static  persistent blocks/SM %d: %.1f GB/s\n", bps, N4 * 20.0 / ms / 1e6);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
