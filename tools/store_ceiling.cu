// store_ceiling.cu — microbenchmark of the output path of the forward kernel:
// how fast can an SM push the 4 GiB int32 coefficient stream of config 2 to
// HBM with (a) TMA tensor stores of P row pairs (box {32, 32 blocks, P, 1},
// 128B swizzle, the 4-D view used by fwd_kernel), (b) 1-D bulk copies of a
// whole 32 KB tile, (c) plain coalesced st.global.v4 from registers.
// No compute: the staging buffers hold garbage.  Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/sc tools/store_ceiling.cu && /tmp/sc
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../paper_1606_05562_b200/csrc/ptx.cuh"

using namespace dct16a;

constexpr long long kBlocks = 4096LL * 1024;   // config 2
constexpr int kTiles = kBlocks / 32;

__device__ __forceinline__ void bulk_s2g(void* g, const void* s, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g), "r"(smem_addr(s)),
                 "r"(bytes)
                 : "memory");
}

template <int P, int BUFS>
__global__ void tma_store_kernel(const __grid_constant__ CUtensorMap tout, int warps) {
    extern __shared__ uint8_t sm[];
    uint8_t* base = sm + ((1024u - (smem_addr(sm) & 1023u)) & 1023u);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint8_t* buf = base + warp * BUFS * P * 4096;
    const long long gw = blockIdx.x * (long long)warps + warp, nw = gridDim.x * (long long)warps;
    int ob = 0;
    for (long long t = gw; t < kTiles; t += nw) {
        const int strip = (int)(t / 1);   // 32 blocks per strip (BX = 32)
        for (int r = 0; r < 8; r += P) {
            if (lane == 0) bulk_wait_read<BUFS - 1>();
            __syncwarp();
            *reinterpret_cast<int4*>(buf + ob * P * 4096 + lane * 16) = make_int4(r, lane, 0, 0);
            fence_async_smem();
            __syncwarp();
            if (lane == 0) {
                tma_store_4d(&tout, buf + ob * P * 4096, 0, 0, r, strip);
                bulk_commit();
            }
            ob = ob + 1 == BUFS ? 0 : ob + 1;
        }
    }
    if (lane == 0) bulk_wait<0>();
}

template <int BUFS>
__global__ void bulk_store_kernel(int32_t* out, int warps) {
    extern __shared__ uint8_t sm[];
    uint8_t* base = sm + ((1024u - (smem_addr(sm) & 1023u)) & 1023u);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint8_t* buf = base + warp * BUFS * 32768;
    const long long gw = blockIdx.x * (long long)warps + warp, nw = gridDim.x * (long long)warps;
    int ob = 0;
    for (long long t = gw; t < kTiles; t += nw) {
        if (lane == 0) bulk_wait_read<BUFS - 1>();
        __syncwarp();
        *reinterpret_cast<int4*>(buf + ob * 32768 + lane * 16) = make_int4(1, lane, 0, 0);
        fence_async_smem();
        __syncwarp();
        if (lane == 0) {
            bulk_s2g(out + t * 8192, buf + ob * 32768, 32768);
            bulk_commit();
        }
        ob = ob + 1 == BUFS ? 0 : ob + 1;
    }
    if (lane == 0) bulk_wait<0>();
}

__global__ void stg_kernel(int32_t* out) {
    const int lane = threadIdx.x & 31;
    const long long gw = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nw = (gridDim.x * (long long)blockDim.x) >> 5;
    for (long long t = gw; t < kTiles; t += nw) {
        int4* dst = reinterpret_cast<int4*>(out + t * 8192);
#pragma unroll 8
        for (int i = 0; i < 64; ++i) __stcs(dst + i * 32 + lane, make_int4(i, lane, 0, 0));
    }
}


// ---- read+write mix of config 2: TMA-load a 16x512 u8 tile (8 KB), write 32 KB
template <int P, int BUFS, int STAGES, bool LSU, int SCAT = 0>
__global__ void mix_kernel(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout,
                           int32_t* out, int warps) {
    extern __shared__ uint8_t sm[];
    uint8_t* base = sm + ((1024u - (smem_addr(sm) & 1023u)) & 1023u);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wbytes = STAGES * 8192 + BUFS * P * 4096;
    uint8_t* in = base + warp * wbytes;
    uint8_t* buf = in + STAGES * 8192;
    uint64_t* bars = reinterpret_cast<uint64_t*>(base + warps * wbytes) + warp * STAGES;
    const long long gw = blockIdx.x * (long long)warps + warp, nw = gridDim.x * (long long)warps;
    if (lane == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
        for (int s = 0; s < STAGES; ++s) {
            long long t = gw + s * nw;
            if (t < kTiles) {
                mbar_arrive_expect_tx(&bars[s], 8192);
                tma_load_3d(in + s * 8192, &tin, &bars[s], 0, (int)(t % 32) * 16, (int)(t / 32), 0);
                tma_load_3d(in + s * 8192 + 4096, &tin, &bars[s], 256, (int)(t % 32) * 16, (int)(t / 32), 0);
            }
        }
    }
    __syncwarp();
    int ob = 0, it = 0;
    for (long long t = gw; t < kTiles; t += nw, ++it) {
        const int s = it % STAGES;
        mbar_wait(&bars[s], (it / STAGES) & 1);
        int4 v = *reinterpret_cast<const int4*>(in + s * 8192 + lane * 16);
        __syncwarp();
        if (lane == 0) {
            long long nt = t + STAGES * nw;
            if (nt < kTiles) {
                mbar_arrive_expect_tx(&bars[s], 8192);
                tma_load_3d(in + s * 8192, &tin, &bars[s], 0, (int)(nt % 32) * 16, (int)(nt / 32), 0);
                tma_load_3d(in + s * 8192 + 4096, &tin, &bars[s], 256, (int)(nt % 32) * 16, (int)(nt / 32), 0);
            }
        }
        for (int r = 0; r < 8; r += P) {
            if (SCAT == 256) {
                // thread-per-block: row pairs r..r+P-1 of this lane's block, 32 B per store
                int* dst = out + (t * 32 + lane) * 256 + r * 32;
#pragma unroll
                for (int i = 0; i < 4 * P; ++i)
                    asm volatile("st.global.L1::no_allocate.v8.b32 [%0], {%1,%2,%3,%4,%1,%2,%3,%4};" ::"l"(dst + i * 8),
                                 "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
            } else if (SCAT == 128) {
                int4* dst = reinterpret_cast<int4*>(out + (t * 32 + lane) * 256 + r * 32);
#pragma unroll
                for (int i = 0; i < 8 * P; ++i) __stcs(dst + i, v);
            } else if (LSU) {
                int4* dst = reinterpret_cast<int4*>(out + t * 8192) + lane;
#pragma unroll
                for (int i = 0; i < 8 * P; ++i) __stcs(dst + (r * 8 + i) * 32, v);
            } else {
                if (lane == 0) bulk_wait_read<BUFS - 1>();
                __syncwarp();
                *reinterpret_cast<int4*>(buf + ob * P * 4096 + lane * 16) = v;
                fence_async_smem();
                __syncwarp();
                if (lane == 0) {
                    tma_store_4d(&tout, buf + ob * P * 4096, 0, 0, r, (int)t);
                    bulk_commit();
                }
                ob = ob + 1 == BUFS ? 0 : ob + 1;
            }
        }
    }
    if (lane == 0) bulk_wait<0>();
}

struct MixCtx {
    CUtensorMap tin, tout[4];
    int32_t* out;
    int sms, warps;
};

template <int P, int BUFS, int STAGES, bool LSU, int SCAT = 0>
static void run_mix(MixCtx* c) {
    const int wbytes = STAGES * 8192 + BUFS * P * 4096;
    const int smem = 1024 + c->warps * (wbytes + STAGES * 8);
    cudaFuncSetAttribute(mix_kernel<P, BUFS, STAGES, LSU, SCAT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int per_sm = 227 * 1024 / smem;
    if (per_sm < 1) per_sm = 1;
    mix_kernel<P, BUFS, STAGES, LSU, SCAT><<<c->sms * per_sm, c->warps * 32, smem>>>(
        c->tin, c->tout[P == 1 ? 0 : P == 2 ? 1 : P == 4 ? 2 : 3], c->out, c->warps);
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static float time_it(void (*launch)(void*), void* arg) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 3; ++i) launch(arg);
    cudaEventRecord(a);
    for (int i = 0; i < 20; ++i) launch(arg);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / 20;
}

struct Ctx {
    CUtensorMap maps[4];
    int32_t* out;
    int sms;
    int mode, warps;
};

template <int P, int BUFS>
static void run_tma(Ctx* c) {
    const int smem = 1024 + c->warps * BUFS * P * 4096;
    cudaFuncSetAttribute(tma_store_kernel<P, BUFS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int per_sm = 227 * 1024 / smem;
    if (per_sm < 1) per_sm = 1;
    tma_store_kernel<P, BUFS><<<c->sms * per_sm, c->warps * 32, smem>>>(c->maps[P == 1 ? 0 : P == 2 ? 1 : P == 4 ? 2 : 3], c->warps);
}

int main() {
    Ctx c;
    cudaDeviceGetAttribute(&c.sms, cudaDevAttrMultiProcessorCount, 0);
    cudaMalloc(&c.out, kBlocks * 1024);
    void* fp;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    EncodeFn enc = (EncodeFn)fp;
    const int Ps[4] = {1, 2, 4, 8};
    for (int i = 0; i < 4; ++i) {
        cuuint64_t dims[4] = {32, 32, 8, (cuuint64_t)kTiles};
        cuuint64_t strides[3] = {1024, 128, 32 * 1024};
        cuuint32_t box[4] = {32, 32, (cuuint32_t)Ps[i], 1};
        cuuint32_t es[4] = {1, 1, 1, 1};
        CUresult r = enc(&c.maps[i], CU_TENSOR_MAP_DATA_TYPE_INT32, 4, c.out, dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r) printf("encode %d failed %d\n", i, r);
    }
    const double bytes = kBlocks * 1024.0;
    auto report = [&](const char* name, float ms) {
        printf("%-34s %8.3f ms  %8.1f GB/s (write only)\n", name, ms, bytes / ms / 1e6);
    };
#define TMA(P, B, W)                                                                        \
    {                                                                                       \
        c.warps = W;                                                                        \
        float ms = time_it([](void* a) { run_tma<P, B>((Ctx*)a); }, &c);                   \
        char nm[64];                                                                        \
        snprintf(nm, 64, "tma P=%d bufs=%d warps/cta=%d", P, B, W);                         \
        report(nm, ms);                                                                     \
    }
    TMA(8, 1, 4)
    for (int W : {2, 3, 4, 6}) {
        c.warps = W;
        float ms = time_it(
            [](void* a) {
                Ctx* c = (Ctx*)a;
                const int smem = 1024 + c->warps * 2 * 32768;
                cudaFuncSetAttribute(bulk_store_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                int per_sm = 227 * 1024 / smem;
                if (per_sm < 1) per_sm = 1;
                bulk_store_kernel<2><<<c->sms * per_sm, c->warps * 32, smem>>>(c->out, c->warps);
            },
            &c);
        char nm[64];
        snprintf(nm, 64, "bulk 32KB bufs=2 warps/cta=%d", W);
        report(nm, ms);
    }
    for (int tpb : {128, 256, 512}) {
        c.warps = tpb;
        float ms = time_it(
            [](void* a) {
                Ctx* c = (Ctx*)a;
                stg_kernel<<<c->sms * (2048 / c->warps), c->warps>>>(c->out);
            },
            &c);
        char nm[64];
        snprintf(nm, 64, "stg.v4 full occupancy tpb=%d", tpb);
        report(nm, ms);
    }
    for (int wps : {4, 8, 16}) {
        c.warps = wps;
        float ms = time_it(
            [](void* a) {
                Ctx* c = (Ctx*)a;
                stg_kernel<<<c->sms, c->warps * 32>>>(c->out);
            },
            &c);
        char nm[64];
        snprintf(nm, 64, "stg.v4 %d warps/SM", wps);
        report(nm, ms);
    }

    {
        MixCtx m;
        m.sms = c.sms;
        m.out = c.out;
        for (int i = 0; i < 4; ++i) m.tout[i] = c.maps[i];
        uint8_t* in;
        cudaMalloc(&in, 4096LL * 512 * 512);
        cudaMemset(in, 1, 4096LL * 512 * 512);
        cuuint64_t dims[3] = {512, 512, 4096};
        cuuint64_t strides[2] = {512, 512 * 512};
        cuuint32_t box[3] = {256, 16, 1};
        cuuint32_t es[3] = {1, 1, 1};
        enc(&m.tin, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, in, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        const double mb = kBlocks * 1280.0;
        auto rep = [&](const char* name, float ms) { printf("%-40s %8.3f ms  %8.1f GB/s (r+w mix)\n", name, ms, mb / ms / 1e6); };
#define MIX(P, B, S, L, W)                                                           \
        {                                                                            \
            m.warps = W;                                                             \
            float ms = time_it([](void* a) { run_mix<P, B, S, L>((MixCtx*)a); }, &m); \
            char nm[80];                                                             \
            snprintf(nm, 80, "mix P=%d bufs=%d stages=%d lsu=%d warps=%d", P, B, S, (int)L, W); \
            rep(nm, ms);                                                             \
        }
#define MIXS(S, W, SC)                                                                       \
        {                                                                                    \
            m.warps = W;                                                                     \
            float ms = time_it([](void* a) { run_mix<1, 1, S, true, SC>((MixCtx*)a); }, &m); \
            char nm[80];                                                                     \
            snprintf(nm, 80, "mix scattered%d stages=%d warps=%d", SC, S, W);                \
            rep(nm, ms);                                                                     \
        }
        MIX(4, 2, 2, false, 4) MIX(8, 1, 2, false, 4)
        MIX(1, 1, 3, true, 4) MIX(1, 1, 2, true, 8)
        MIXS(2, 4, 256) MIXS(3, 4, 256) MIXS(4, 4, 256) MIXS(2, 8, 256) MIXS(3, 4, 128) MIXS(2, 8, 128)
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
