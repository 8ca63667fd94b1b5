// alu_rates.cu — per-SM issue rates of the arithmetic the codec kernels use
// (FP64 add/fma, FP32 add/fma, INT32 add, conversions), measured on the box.
// Each thread runs 8 independent dependency chains so latency is hidden; the
// rate is ops / (SMs · cycles) with cycles from clock64 on SM 0.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/alu_rates tools/alu_rates.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

template <int OP>
__global__ void __launch_bounds__(256) k(float* outf, double* outd, int* outi, long long* cyc, float sf, double sd, int si) {
    long long t0 = clock64();
    if constexpr (OP == 0) {  // DADD
        double a[8];
        for (int j = 0; j < 8; ++j) a[j] = threadIdx.x + j;
#pragma unroll 16
        for (int i = 0; i < ITERS; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) a[j] = a[j] + sd;
        double s = 0; for (int j = 0; j < 8; ++j) s += a[j];
        if (s == 12345.0) outd[0] = s;
    } else if constexpr (OP == 1) {  // DFMA
        double a[8];
        for (int j = 0; j < 8; ++j) a[j] = threadIdx.x + j;
#pragma unroll 16
        for (int i = 0; i < ITERS; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) a[j] = fma(a[j], sd, sd);
        double s = 0; for (int j = 0; j < 8; ++j) s += a[j];
        if (s == 12345.0) outd[0] = s;
    } else if constexpr (OP == 2) {  // FADD reg-reg
        float a[8];
        for (int j = 0; j < 8; ++j) a[j] = threadIdx.x + j;
#pragma unroll 16
        for (int i = 0; i < ITERS; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) a[j] = a[j] + sf;
        float s = 0; for (int j = 0; j < 8; ++j) s += a[j];
        if (s == 12345.f) outf[0] = s;
    } else if constexpr (OP == 3) {  // FADD a+b with both variable (a[j] + a[j+1])
        float a[8];
        for (int j = 0; j < 8; ++j) a[j] = threadIdx.x + j;
#pragma unroll 16
        for (int i = 0; i < ITERS; ++i) {
#pragma unroll
            for (int j = 0; j < 8; ++j) a[j] = a[j] + a[(j + 1) & 7];
        }
        float s = 0; for (int j = 0; j < 8; ++j) s += a[j];
        if (s == 12345.f) outf[0] = s;
    } else if constexpr (OP == 4) {  // IADD (2-input, variable)
        int a[8];
        for (int j = 0; j < 8; ++j) a[j] = threadIdx.x + j;
#pragma unroll 16
        for (int i = 0; i < ITERS; ++i) {
#pragma unroll
            for (int j = 0; j < 8; ++j) a[j] = a[j] + a[(j + 1) & 7];
        }
        int s = 0; for (int j = 0; j < 8; ++j) s += a[j];
        if (s == 12345) outi[0] = s;
    } else if constexpr (OP == 5) {  // DADD variable
        double a[8];
        for (int j = 0; j < 8; ++j) a[j] = threadIdx.x + j;
#pragma unroll 16
        for (int i = 0; i < ITERS; ++i) {
#pragma unroll
            for (int j = 0; j < 8; ++j) a[j] = a[j] + a[(j + 1) & 7];
        }
        double s = 0; for (int j = 0; j < 8; ++j) s += a[j];
        if (s == 12345.0) outd[0] = s;
    } else if constexpr (OP == 6) {  // mixed: 1 IADD + 1 FADD + 1 DADD per step
        int ai[4]; float af[4]; double ad[4];
        for (int j = 0; j < 4; ++j) { ai[j] = threadIdx.x + j; af[j] = ai[j]; ad[j] = ai[j]; }
#pragma unroll 16
        for (int i = 0; i < ITERS; ++i) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                ai[j] = ai[j] + ai[(j + 1) & 3];
                af[j] = af[j] + af[(j + 1) & 3];
                ad[j] = ad[j] + ad[(j + 1) & 3];
            }
        }
        double s = 0; for (int j = 0; j < 4; ++j) s += ai[j] + af[j] + ad[j];
        if (s == 12345.0) outd[0] = s;
    } else if constexpr (OP == 7) {  // I2F.F64
        double a[8];
        int x = threadIdx.x;
        for (int j = 0; j < 8; ++j) a[j] = 0;
#pragma unroll 16
        for (int i = 0; i < ITERS; ++i) {
#pragma unroll
            for (int j = 0; j < 8; ++j) a[j] = static_cast<double>(x + i * 8 + j);
            x ^= __double2hiint(a[0]) ^ __double2hiint(a[1]) ^ __double2hiint(a[2]) ^ __double2hiint(a[3]) ^ __double2hiint(a[4]) ^ __double2hiint(a[5]) ^ __double2hiint(a[6]) ^ __double2hiint(a[7]);
        }
        if (x == 12345) outi[0] = x;
    } else if constexpr (OP == 8) {  // I2F.F32
        float a[8];
        int x = threadIdx.x;
#pragma unroll 16
        for (int i = 0; i < ITERS; ++i) {
#pragma unroll
            for (int j = 0; j < 8; ++j) a[j] = static_cast<float>(x + j);
            x ^= __float_as_int(a[0]) ^ __float_as_int(a[1]) ^ __float_as_int(a[2]) ^ __float_as_int(a[3]) ^ __float_as_int(a[4]) ^ __float_as_int(a[5]) ^ __float_as_int(a[6]) ^ __float_as_int(a[7]);
        }
        if (x == 12345) outi[0] = x;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

template <int OP>
void run(const char* name, int sms, double ops_per_thread) {
    float* f; double* d; int* i; long long* c;
    cudaMalloc(&f, 16); cudaMalloc(&d, 16); cudaMalloc(&i, 16); cudaMalloc(&c, 16);
    for (int bpsm : {4, 8}) {
        int grid = sms * bpsm;
        k<OP><<<grid, 256>>>(f, d, i, c, 1.0001f, 1.0000001, 3);
        cudaEvent_t a, b;
        cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a);
        k<OP><<<grid, 256>>>(f, d, i, c, 1.0001f, 1.0000001, 3);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        long long cyc; cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
        double ops = double(grid) * 256 * ops_per_thread;
        // effective clock from cycles of block 0 vs elapsed (block 0 runs the whole time when bpsm fits)
        double ghz = cyc / (ms * 1e6);
        double per_sm_clk = ops / (ms * 1e-3) / sms / (ghz * 1e9);
        printf("%-28s blocks/SM %d  %8.3f ms  %.2f Gop/s  clk~%.2f GHz  ops/SM/clk %.1f\n", name, bpsm, ms,
               ops / (ms * 1e-3) / 1e9, ghz, per_sm_clk);
    }
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    printf("SMs %d\n", sms);
    run<0>("DADD reg+const", sms, 8.0 * ITERS);
    run<1>("DFMA", sms, 8.0 * ITERS);
    run<2>("FADD reg+const", sms, 8.0 * ITERS);
    run<3>("FADD reg+reg", sms, 8.0 * ITERS);
    run<4>("IADD reg+reg", sms, 8.0 * ITERS);
    run<5>("DADD reg+reg", sms, 8.0 * ITERS);
    run<6>("mixed I+F+D (per op)", sms, 12.0 * ITERS);
    run<7>("I2F.F64 (+1 xor)", sms, 8.0 * ITERS);
    run<8>("I2F.F32 (+1 xor)", sms, 8.0 * ITERS);
    return 0;
}
