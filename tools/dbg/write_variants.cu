#include <cstdio>
#include <cuda_runtime.h>
constexpr long long N4 = 4096LL * 512 * 512 / 4;   // int4 elements of 4 GiB
template <int MODE>
__global__ void w(int4* __restrict__ out, long long n, int salt) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride) {
        int4 v = (MODE & 2) ? make_int4(7, 7, 7, 7) : make_int4((int)i ^ salt, (int)(i >> 7) * 33, (int)i * 5 + 1, (int)i * 9 + salt);
        if (MODE & 1) __stcs(out + i, v); else out[i] = v;
    }
}
template <class F> float timeit(F f) {
    f(); cudaDeviceSynchronize(); cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a); for (int r = 0; r < 20; ++r) f(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); return ms / 20;
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int4* out; cudaMalloc(&out, N4 * 16);
    const char* names[4] = {"plain, varying", "stcs, varying", "plain, constant", "stcs, constant"};
    for (int bps : {2, 4, 8}) {
        int grid = sms * bps;
        float ms[4] = {timeit([&]{ w<0><<<grid, 256>>>(out, N4, 3); }), timeit([&]{ w<1><<<grid, 256>>>(out, N4, 3); }),
                       timeit([&]{ w<2><<<grid, 256>>>(out, N4, 3); }), timeit([&]{ w<3><<<grid, 256>>>(out, N4, 3); })};
        for (int m = 0; m < 4; ++m) printf("blocks/SM %d tpb 256 %-16s %.3f ms %.1f GB/s\n", bps, names[m], ms[m], N4 * 16.0 / ms[m] / 1e6);
    }
    float ms = timeit([&]{ cudaMemsetAsync(out, 0, N4 * 16); });
    printf("cudaMemset 4 GiB %.3f ms %.1f GB/s\n", ms, N4 * 16.0 / ms / 1e6);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
