// abi.cu — the C ABI of include/dct16a.h: argument validation (synchronous,
// before any launch), error codes, thread-local error text, tensor-map
// encoding through the driver entry point, and dispatch to the launchers.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>

#include <atomic>
#include <mutex>
#include <stdlib.h>

#include "internal.h"
#include "sched.cuh"

namespace dct16a {
namespace {

thread_local char g_err[512] = "";

int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Validate a descriptor and fill the geometry.  Reading of the shape/pitch rules:
// SURVEY.md §8(b) conventions, restated in include/dct16a.h.
int check_desc(const dct16a_desc* d, Geom* g) {
    if (!d) return fail(DCT16A_ENULL, "desc is NULL");
    if (d->bit_depth != 8 && d->bit_depth != 10)
        return fail(DCT16A_EDOMAIN, "bit_depth %d not in {8, 10}", d->bit_depth);
    if (d->width <= 0 || d->height <= 0 || (d->width % 16) || (d->height % 16))
        return fail(DCT16A_ESHAPE, "width %d / height %d must be positive multiples of 16", d->width,
                    d->height);
    if (d->batch < 1) return fail(DCT16A_ESHAPE, "batch %d < 1", d->batch);
    if (d->valid_height <= 0 || d->valid_height > d->height)
        return fail(DCT16A_ESHAPE, "valid_height %d outside (0, %d]", d->valid_height, d->height);
    if (d->reserved != 0) return fail(DCT16A_EDOMAIN, "desc.reserved must be 0");
    const int elem = d->bit_depth == 8 ? 1 : 2;
    if (d->pitch_bytes < static_cast<int64_t>(d->width) * elem || (d->pitch_bytes % 16))
        return fail(DCT16A_EPITCH, "pitch %lld must be >= width*elem and a multiple of 16",
                    static_cast<long long>(d->pitch_bytes));
    if (d->image_stride_bytes % 16)
        return fail(DCT16A_EPITCH, "image_stride %lld not a multiple of 16",
                    static_cast<long long>(d->image_stride_bytes));
    if (d->batch > 1 && d->image_stride_bytes < d->pitch_bytes * d->height)
        return fail(DCT16A_EPITCH, "image_stride %lld < pitch*height",
                    static_cast<long long>(d->image_stride_bytes));
    if (d->pitch_bytes >= (int64_t(1) << 40) || d->image_stride_bytes >= (int64_t(1) << 40))
        return fail(DCT16A_EPITCH, "pitch/stride too large for a tensor map");
    g->W = d->width;
    g->H = d->height;
    g->VH = d->valid_height;
    g->N = d->batch;
    g->bits = d->bit_depth;
    g->BX = d->width / 16;
    g->BY = d->height / 16;
    g->elem = elem;
    g->pitch = d->pitch_bytes;
    g->istride = d->batch > 1 ? d->image_stride_bytes
                              : (d->image_stride_bytes > 0 ? d->image_stride_bytes
                                                           : d->pitch_bytes * d->height);
    g->nblocks = static_cast<int64_t>(g->N) * g->BX * g->BY;
    return 0;
}

int check_quant(const dct16a_quant* q) {
    if (!q) return fail(DCT16A_ENULL, "quant is NULL");
    if (q->reserved != 0) return fail(DCT16A_EDOMAIN, "quant.reserved must be 0");
    if (q->mode == DCT16A_ZONAL) {
        if (q->r < 1 || q->r > 256) return fail(DCT16A_EDOMAIN, "r=%d outside [1, 256]", q->r);
    } else if (q->mode == DCT16A_UNIFORM) {
        if (q->step < 1 || q->step > 65535)
            return fail(DCT16A_EDOMAIN, "step=%d outside [1, 65535]", q->step);
    } else {
        return fail(DCT16A_EDOMAIN, "unknown quantiser mode %d", q->mode);
    }
    return 0;
}

// Byte extent of an image batch in memory: [p, p + extent).
int64_t image_extent(const Geom& g) {
    return static_cast<int64_t>(g.N - 1) * g.istride + static_cast<int64_t>(g.H - 1) * g.pitch +
           static_cast<int64_t>(g.W) * g.elem;
}

bool overlaps(const void* a, int64_t na, const void* b, int64_t nb) {
    const uintptr_t x = reinterpret_cast<uintptr_t>(a), y = reinterpret_cast<uintptr_t>(b);
    return x < y + static_cast<uintptr_t>(nb) && y < x + static_cast<uintptr_t>(na);
}

int check_ptr(const void* p, const char* name) {
    if (!p) return fail(DCT16A_ENULL, "%s is NULL", name);
    if (!aligned16(p)) return fail(DCT16A_EALIGN, "%s is not 16-byte aligned", name);
    return 0;
}

int launched(int rc, const char* what) {
    if (rc == 0) {
        g_err[0] = 0;
        return DCT16A_OK;
    }
    if (rc < 0) return fail(rc, "%s: tensor-map encode failed", what);
    return fail(DCT16A_ECUDA, "%s: %s", what, cudaGetErrorString(static_cast<cudaError_t>(rc)));
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn get_encode() {
    static EncodeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    });
    return fn;
}

}  // namespace

int encode_tiled(CUtensorMap* map, CUtensorMapDataType dt, uint32_t rank, const void* gaddr,
                 const uint64_t* dims, const uint64_t* strides_bytes, const uint32_t* box,
                 CUtensorMapSwizzle swz, CUtensorMapL2promotion promo) {
    EncodeFn fn = get_encode();
    if (!fn) return -1;
    cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    CUresult r = fn(map, dt, rank, const_cast<void*>(gaddr), reinterpret_cast<const cuuint64_t*>(dims),
                    reinterpret_cast<const cuuint64_t*>(strides_bytes), reinterpret_cast<const cuuint32_t*>(box),
                    estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz, promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return static_cast<int>(r);
}

namespace {
int env_int(const char* name, int dflt) {
    const char* e = getenv(name);
    return e ? atoi(e) : dflt;
}
// The product build ships codec paths 0 and 2 and forward store modes 3 and 5
// (the defaults); -DDCT16A_EXPERIMENTS adds the round-1 variants.
bool codec_path_built(int v) {
#ifdef DCT16A_EXPERIMENTS
    return v >= 0 && v <= 4;
#else
    return v == 0 || v == 2;
#endif
}
bool store_mode_built(int v) {
#ifdef DCT16A_EXPERIMENTS
    return v >= -1 && v <= 7;
#else
    return v == -1 || v == 3 || v == 5;
#endif
}
int env_option(const char* name, int dflt, bool (*ok)(int)) {
    const int v = env_int(name, dflt);
    return ok(v) ? v : dflt;   // an unbuilt value in the environment falls back to the default
}
std::atomic<int> g_codec_path{env_option("DCT16A_CODEC_PATH", 0, codec_path_built)};
std::atomic<int> g_fwd_store{env_option("DCT16A_FWD_STORE", -1, store_mode_built)};
bool uniform_quant_valid(int v) { return v >= 0 && v <= 2; }
std::atomic<int> g_uniform_quant{env_option("DCT16A_UNIFORM_QUANT", 0, uniform_quant_valid)};
}  // namespace

int get_option(int option) {
    if (option == DCT16A_OPT_CODEC_PATH) return g_codec_path.load(std::memory_order_relaxed);
    if (option == DCT16A_OPT_FWD_STORE) return g_fwd_store.load(std::memory_order_relaxed);
    if (option == DCT16A_OPT_UNIFORM_QUANT) return g_uniform_quant.load(std::memory_order_relaxed);
    return 0;
}

int smem_optin(const void* func, int bytes) {
    int dev = 0;
    cudaGetDevice(&dev);
    static std::mutex mu;
    static struct Entry {
        const void* f;
        uint64_t devmask;
    } done[64];
    static int n_done = 0;
    std::lock_guard<std::mutex> lock(mu);
    int i = 0;
    while (i < n_done && done[i].f != func) ++i;
    if (i < n_done && dev < 64 && ((done[i].devmask >> dev) & 1u)) return 0;
    const cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e) return static_cast<int>(e);
    if (i == n_done && n_done < 64) done[n_done++] = {func, 0};
    if (i < n_done && dev < 64) done[i].devmask |= uint64_t(1) << dev;
    return 0;
}

// ---- tile-scheduler slots (sched.cuh, SchedGuard in internal.h)
namespace {
struct SlotTable {
    std::mutex mu;
    unsigned seq = 0;
    cudaEvent_t ev[kSchedSlots] = {};
    cudaStream_t st[kSchedSlots] = {};
    bool used[kSchedSlots] = {};
};
constexpr int kMaxDevices = 64;
SlotTable* slot_table(int family, int dev) {
    static std::mutex mu;
    static SlotTable* tables[kSchedFamilies][kMaxDevices] = {};
    std::lock_guard<std::mutex> lock(mu);
    SlotTable*& t = tables[family][dev];
    if (!t) t = new SlotTable();   // one per (family, device), never freed
    return t;
}
}  // namespace

SchedGuard::SchedGuard(int family, cudaStream_t st) : st_(st) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) {
        err_ = static_cast<int>(cudaGetLastError());
        if (!err_) err_ = static_cast<int>(cudaErrorInvalidDevice);
        return;
    }
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess) {
        (void)cudaGetLastError();   // e.g. the legacy stream during another thread's global capture
        cs = cudaStreamCaptureStatusActive;
    }
    if (cs != cudaStreamCaptureStatusNone) return;   // captured: static schedule, no shared counter
    SlotTable* t = slot_table(family, dev);
    t->mu.lock();
    state_ = t;
    const int s = static_cast<int>(t->seq++ % kSchedSlots);
    if (t->used[s] && t->st[s] != st) {
        // the slot's previous launch ran on another stream: order this launch after it
        const cudaError_t q = cudaEventQuery(t->ev[s]);
        if (q == cudaErrorNotReady) {
            err_ = static_cast<int>(cudaStreamWaitEvent(st, t->ev[s], 0));
        } else if (q != cudaSuccess) {
            err_ = static_cast<int>(q);
        }
    }
    slot_ = s;
}

SchedGuard::~SchedGuard() {
    if (!state_) return;
    SlotTable* t = static_cast<SlotTable*>(state_);
    const int s = slot_;
    bool ok = t->ev[s] != nullptr || cudaEventCreateWithFlags(&t->ev[s], cudaEventDisableTiming) == cudaSuccess;
    if (ok) ok = cudaEventRecord(t->ev[s], st_) == cudaSuccess;
    if (ok) {
        t->st[s] = st_;
        t->used[s] = true;
    } else {
        // no completion event: make every later user of this slot wait for the device
        (void)cudaGetLastError();
        cudaStreamSynchronize(st_);
        t->used[s] = false;
    }
    t->mu.unlock();
}

int num_sms() {
    int dev = 0;
    cudaGetDevice(&dev);
    static int cache[64] = {0};
    if (dev >= 0 && dev < 64 && cache[dev]) return cache[dev];
    int n = 148;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (dev >= 0 && dev < 64) cache[dev] = n;
    return n;
}

}  // namespace dct16a

using namespace dct16a;

extern "C" {

DCT16A_API int dct16a_forward(const void* src, const dct16a_desc* desc, int32_t* coef, void* stream) {
    Geom g;
    int rc;
    if ((rc = check_desc(desc, &g))) return rc;
    if ((rc = check_ptr(src, "src")) || (rc = check_ptr(coef, "coef"))) return rc;
    if (overlaps(coef, g.nblocks * 1024, src, image_extent(g))) return fail(DCT16A_EDOMAIN, "coef overlaps src");
    return launched(launch_forward(src, g, coef, static_cast<cudaStream_t>(stream)), "dct16a_forward");
}

DCT16A_API int dct16a_forward16(const void* src, const dct16a_desc* desc, int16_t* coef16, void* stream) {
    Geom g;
    int rc;
    if ((rc = check_desc(desc, &g))) return rc;
    if (g.bits != 8) return fail(DCT16A_EDOMAIN, "dct16a_forward16 needs 8-bit images (10-bit Z exceeds 16 bits)");
    if ((rc = check_ptr(src, "src")) || (rc = check_ptr(coef16, "coef16"))) return rc;
    return launched(launch_forward16(src, g, coef16, static_cast<cudaStream_t>(stream)), "dct16a_forward16");
}

DCT16A_API int dct16a_quantize(const int32_t* coef, const dct16a_desc* desc, const dct16a_quant* quant,
                               int32_t* qcoef, float* scaled, void* stream) {
    Geom g;
    int rc;
    if ((rc = check_desc(desc, &g)) || (rc = check_quant(quant))) return rc;
    if ((rc = check_ptr(coef, "coef")) || (rc = check_ptr(qcoef, "qcoef"))) return rc;
    if (scaled && !aligned16(scaled)) return fail(DCT16A_EALIGN, "scaled is not 16-byte aligned");
    return launched(launch_quantize(coef, g, *quant, qcoef, scaled, static_cast<cudaStream_t>(stream)),
                    "dct16a_quantize");
}

DCT16A_API int dct16a_inverse(const int32_t* qcoef, const dct16a_desc* desc, const dct16a_quant* quant,
                              void* recon, void* stream) {
    Geom g;
    int rc;
    if ((rc = check_desc(desc, &g)) || (rc = check_quant(quant))) return rc;
    if ((rc = check_ptr(qcoef, "qcoef")) || (rc = check_ptr(recon, "recon"))) return rc;
    return launched(launch_inverse(qcoef, g, *quant, recon, static_cast<cudaStream_t>(stream)),
                    "dct16a_inverse");
}

DCT16A_API int dct16a_psnr(const void* ref, const void* test, const dct16a_desc* desc, uint64_t* sse,
                           double* psnr, void* stream) {
    Geom g;
    int rc;
    if ((rc = check_desc(desc, &g))) return rc;
    if ((rc = check_ptr(ref, "ref")) || (rc = check_ptr(test, "test"))) return rc;
    if (!sse) return fail(DCT16A_ENULL, "sse is NULL");
    if (reinterpret_cast<uintptr_t>(sse) & 7u) return fail(DCT16A_EALIGN, "sse is not 8-byte aligned");
    if (psnr && (reinterpret_cast<uintptr_t>(psnr) & 7u)) return fail(DCT16A_EALIGN, "psnr not 8-byte aligned");
    if (static_cast<long long>(g.VH) * g.W * g.elem / 16 >= (1LL << 31))
        return fail(DCT16A_ESHAPE, "valid_height*width*elem = %lld bytes per image: dct16a_psnr takes < 32 GiB",
                    static_cast<long long>(g.VH) * g.W * g.elem);
    return launched(launch_psnr(ref, test, g, sse, psnr, static_cast<cudaStream_t>(stream)), "dct16a_psnr");
}

DCT16A_API int dct16a_codec(const void* src, const dct16a_desc* desc, const dct16a_quant* quant, void* recon,
                            uint64_t* sse, double* psnr, void* stream) {
    Geom g;
    int rc;
    if ((rc = check_desc(desc, &g)) || (rc = check_quant(quant))) return rc;
    if ((rc = check_ptr(src, "src"))) return rc;
    if (recon && !aligned16(recon)) return fail(DCT16A_EALIGN, "recon is not 16-byte aligned");
    if (recon && overlaps(recon, image_extent(g), src, image_extent(g)))
        return fail(DCT16A_EDOMAIN, "recon overlaps src (the reconstruction would overwrite unread input)");
    if (!sse) return fail(DCT16A_ENULL, "sse is NULL");
    if (reinterpret_cast<uintptr_t>(sse) & 7u) return fail(DCT16A_EALIGN, "sse is not 8-byte aligned");
    if (psnr && (reinterpret_cast<uintptr_t>(psnr) & 7u)) return fail(DCT16A_EALIGN, "psnr not 8-byte aligned");
    return launched(launch_codec(src, g, *quant, recon, sse, psnr, static_cast<cudaStream_t>(stream)),
                    "dct16a_codec");
}

DCT16A_API int dct16a_codec_allreduce(const void* src, const dct16a_desc* desc, const dct16a_quant* quant,
                                      void* recon, uint64_t* const* sse_peers, int32_t n_peers, int64_t frame_offset,
                                      void* stream) {
    Geom g;
    int rc;
    if ((rc = check_desc(desc, &g)) || (rc = check_quant(quant))) return rc;
    if ((rc = check_ptr(src, "src"))) return rc;
    if (recon && !aligned16(recon)) return fail(DCT16A_EALIGN, "recon is not 16-byte aligned");
    if (recon && overlaps(recon, image_extent(g), src, image_extent(g)))
        return fail(DCT16A_EDOMAIN, "recon overlaps src (the reconstruction would overwrite unread input)");
    if (!sse_peers) return fail(DCT16A_ENULL, "sse_peers is NULL");
    if (n_peers < 1 || n_peers > 8) return fail(DCT16A_EDOMAIN, "n_peers %d outside [1, 8]", n_peers);
    if (frame_offset < 0) return fail(DCT16A_EDOMAIN, "frame_offset %lld < 0", static_cast<long long>(frame_offset));
    for (int i = 0; i < n_peers; ++i) {
        if (!sse_peers[i]) return fail(DCT16A_ENULL, "sse_peers[%d] is NULL", i);
        if (reinterpret_cast<uintptr_t>(sse_peers[i]) & 7u) return fail(DCT16A_EALIGN, "sse_peers[%d] not 8-byte aligned", i);
    }
    return launched(launch_codec_allreduce(src, g, *quant, recon, sse_peers, n_peers, frame_offset, 0,
                                           static_cast<cudaStream_t>(stream)),
                    "dct16a_codec_allreduce");
}

DCT16A_API int dct16a_codec_allreduce_multicast(const void* src, const dct16a_desc* desc, const dct16a_quant* quant,
                                                void* recon, uint64_t* sse_multicast, int64_t frame_offset,
                                                void* stream) {
    Geom g;
    int rc;
    if ((rc = check_desc(desc, &g)) || (rc = check_quant(quant))) return rc;
    if ((rc = check_ptr(src, "src"))) return rc;
    if (recon && !aligned16(recon)) return fail(DCT16A_EALIGN, "recon is not 16-byte aligned");
    if (recon && overlaps(recon, image_extent(g), src, image_extent(g)))
        return fail(DCT16A_EDOMAIN, "recon overlaps src (the reconstruction would overwrite unread input)");
    if (!sse_multicast) return fail(DCT16A_ENULL, "sse_multicast is NULL");
    if (reinterpret_cast<uintptr_t>(sse_multicast) & 7u) return fail(DCT16A_EALIGN, "sse_multicast not 8-byte aligned");
    if (frame_offset < 0) return fail(DCT16A_EDOMAIN, "frame_offset %lld < 0", static_cast<long long>(frame_offset));
    uint64_t* const peers[1] = {sse_multicast};
    return launched(launch_codec_allreduce(src, g, *quant, recon, peers, 1, frame_offset, 1,
                                           static_cast<cudaStream_t>(stream)),
                    "dct16a_codec_allreduce_multicast");
}

DCT16A_API int dct16a_ssim(const void* ref, const void* test, const dct16a_desc* desc, double* ssim,
                           void* stream) {
    Geom g;
    int rc;
    if ((rc = check_desc(desc, &g))) return rc;
    if ((rc = check_ptr(ref, "ref")) || (rc = check_ptr(test, "test"))) return rc;
    if (g.VH < 11) return fail(DCT16A_ESHAPE, "valid_height %d < 11 (SSIM window)", g.VH);
    if (!ssim) return fail(DCT16A_ENULL, "ssim is NULL");
    if (reinterpret_cast<uintptr_t>(ssim) & 7u) return fail(DCT16A_EALIGN, "ssim is not 8-byte aligned");
    return launched(launch_ssim(ref, test, g, ssim, static_cast<cudaStream_t>(stream)), "dct16a_ssim");
}

DCT16A_API int dct16a_zonal_sweep(const void* src, const dct16a_desc* desc, int32_t r_first, int32_t r_count,
                                  uint64_t* sse, double* psnr, void* stream) {
    Geom g;
    int rc;
    if ((rc = check_desc(desc, &g))) return rc;
    if ((rc = check_ptr(src, "src"))) return rc;
    if (r_first < 1 || r_count < 1 || r_first + r_count - 1 > 256)
        return fail(DCT16A_EDOMAIN, "r range [%d, %d] outside [1, 256]", r_first, r_first + r_count - 1);
    if (!sse) return fail(DCT16A_ENULL, "sse is NULL");
    if (reinterpret_cast<uintptr_t>(sse) & 7u) return fail(DCT16A_EALIGN, "sse is not 8-byte aligned");
    if (psnr && (reinterpret_cast<uintptr_t>(psnr) & 7u)) return fail(DCT16A_EALIGN, "psnr not 8-byte aligned");
    return launched(launch_sweep(src, g, r_first, r_count, sse, psnr, static_cast<cudaStream_t>(stream)),
                    "dct16a_zonal_sweep");
}

DCT16A_API int dct16a_sse_psnr(const uint64_t* sse, int64_t count, const dct16a_desc* desc, double* psnr,
                               uint64_t* sse_total, double* psnr_total, void* stream) {
    Geom g;
    int rc;
    if ((rc = check_desc(desc, &g))) return rc;
    if (!sse) return fail(DCT16A_ENULL, "sse is NULL");
    if (count < 1 || count > (int64_t(1) << 31) - 1)
        return fail(DCT16A_ESHAPE, "count %lld outside [1, 2^31)", static_cast<long long>(count));
    if (reinterpret_cast<uintptr_t>(sse) & 7u) return fail(DCT16A_EALIGN, "sse is not 8-byte aligned");
    for (const void* p : {static_cast<const void*>(psnr), static_cast<const void*>(sse_total),
                          static_cast<const void*>(psnr_total)})
        if (p && (reinterpret_cast<uintptr_t>(p) & 7u)) return fail(DCT16A_EALIGN, "an output is not 8-byte aligned");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    rc = launch_psnr_finish(g, count, const_cast<uint64_t*>(sse), psnr, st);
    if (!rc) rc = launch_sse_total(g, count, sse, sse_total, psnr_total, st);
    return launched(rc, "dct16a_sse_psnr");
}

// ---- end-to-end forward from host buffers (dct16a_forward_host)
namespace {
// The chunk pipeline's two streams and events, created once per device.
struct HostPipe {
    std::mutex mu;
    cudaStream_t s[2] = {};
    cudaEvent_t fork = nullptr, join[2] = {};
    bool ready = false;
};
HostPipe* host_pipe(int dev) {
    static std::mutex mu;
    static HostPipe* pipes[kMaxDevices] = {};
    std::lock_guard<std::mutex> lock(mu);
    if (!pipes[dev]) pipes[dev] = new HostPipe();
    return pipes[dev];
}

int64_t chunk_in_bytes(const Geom& g, int64_t m) {   // device bytes of m images, 1 KB aligned
    const int64_t b = (m - 1) * g.istride + static_cast<int64_t>(g.H - 1) * g.pitch + static_cast<int64_t>(g.W) * g.elem;
    return (b + 1023) & ~int64_t(1023);
}
int64_t chunk_out_bytes(const Geom& g, int64_t m) { return m * g.BX * g.BY * 1024; }
}  // namespace

DCT16A_API int64_t dct16a_forward_host_workspace(const dct16a_desc* desc, int32_t chunk_images) {
    Geom g;
    if (check_desc(desc, &g)) return -1;
    if (chunk_images < 1) return fail(DCT16A_EDOMAIN, "chunk_images %d < 1", chunk_images);
    const int64_t m = chunk_images < g.N ? chunk_images : g.N;
    return 2 * (chunk_in_bytes(g, m) + chunk_out_bytes(g, m));
}

DCT16A_API int dct16a_forward_host(const void* host_src, const dct16a_desc* desc, int32_t* host_coef,
                                   void* workspace, int64_t workspace_bytes, void* stream) {
    Geom g;
    int rc;
    if ((rc = check_desc(desc, &g))) return rc;
    if (!host_src) return fail(DCT16A_ENULL, "host_src is NULL");
    if (!host_coef) return fail(DCT16A_ENULL, "host_coef is NULL");
    if ((rc = check_ptr(workspace, "workspace"))) return rc;
    if (reinterpret_cast<uintptr_t>(workspace) & 1023u) return fail(DCT16A_EALIGN, "workspace is not 1024-byte aligned");
    // the largest chunk whose two buffer slots fit the workspace
    int64_t m = 0;
    for (int64_t lo = 1, hi = g.N; lo <= hi;) {
        const int64_t mid = lo + (hi - lo) / 2;
        if (2 * (chunk_in_bytes(g, mid) + chunk_out_bytes(g, mid)) <= workspace_bytes) {
            m = mid;
            lo = mid + 1;
        } else {
            hi = mid - 1;
        }
    }
    if (m < 1)
        return fail(DCT16A_EDOMAIN, "workspace of %lld bytes < %lld (dct16a_forward_host_workspace with one image)",
                    static_cast<long long>(workspace_bytes), static_cast<long long>(2 * (chunk_in_bytes(g, 1) + chunk_out_bytes(g, 1))));
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices)
        return launched(static_cast<int>(cudaGetLastError()), "dct16a_forward_host");
    HostPipe* hp = host_pipe(dev);
    std::lock_guard<std::mutex> lock(hp->mu);
    auto cu = [&](cudaError_t e) { return launched(static_cast<int>(e), "dct16a_forward_host"); };
    if (!hp->ready) {
        for (int i = 0; i < 2; ++i) {
            if (cudaError_t e = cudaStreamCreateWithFlags(&hp->s[i], cudaStreamNonBlocking)) return cu(e);
            if (cudaError_t e = cudaEventCreateWithFlags(&hp->join[i], cudaEventDisableTiming)) return cu(e);
        }
        if (cudaError_t e = cudaEventCreateWithFlags(&hp->fork, cudaEventDisableTiming)) return cu(e);
        hp->ready = true;
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // fork: both pipeline streams start after the caller's prior work
    if (cudaError_t e = cudaEventRecord(hp->fork, st)) return cu(e);
    for (int i = 0; i < 2; ++i)
        if (cudaError_t e = cudaStreamWaitEvent(hp->s[i], hp->fork, 0)) return cu(e);
    const int64_t in_b = chunk_in_bytes(g, m), out_b = chunk_out_bytes(g, m);
    uint8_t* ws = static_cast<uint8_t*>(workspace);
    const uint8_t* hsrc = static_cast<const uint8_t*>(host_src);
    uint8_t* hdst = reinterpret_cast<uint8_t*>(host_coef);
    int64_t i = 0;
    for (int64_t s0 = 0; s0 < g.N; s0 += m, ++i) {
        // chunk i on stream i % 2 into buffer slot i % 2: the slot's previous
        // chunk (i - 2) ran on the same stream, so its copies are ordered before
        const int k = static_cast<int>(i & 1);
        const int64_t mc = g.N - s0 < m ? g.N - s0 : m;
        Geom gc = g;
        gc.N = static_cast<int>(mc);
        gc.nblocks = mc * g.BX * g.BY;
        uint8_t* din = ws + k * (in_b + out_b);
        int32_t* dout = reinterpret_cast<int32_t*>(din + in_b);
        const int64_t nin = (mc - 1) * g.istride + static_cast<int64_t>(g.H - 1) * g.pitch + static_cast<int64_t>(g.W) * g.elem;
        if (cudaError_t e = cudaMemcpyAsync(din, hsrc + s0 * g.istride, nin, cudaMemcpyHostToDevice, hp->s[k])) return cu(e);
        if ((rc = launch_forward(din, gc, dout, hp->s[k]))) return launched(rc, "dct16a_forward_host");
        if (cudaError_t e = cudaMemcpyAsync(hdst + s0 * g.BX * g.BY * 1024, dout, gc.nblocks * 1024,
                                            cudaMemcpyDeviceToHost, hp->s[k]))
            return cu(e);
    }
    // join: the caller's stream continues after both pipeline streams
    for (int k = 0; k < 2; ++k) {
        if (cudaError_t e = cudaEventRecord(hp->join[k], hp->s[k])) return cu(e);
        if (cudaError_t e = cudaStreamWaitEvent(st, hp->join[k], 0)) return cu(e);
    }
    return launched(0, "dct16a_forward_host");
}

DCT16A_API int dct16a_set_option(int option, int value) {
    if (option == DCT16A_OPT_CODEC_PATH) {
        if (!codec_path_built(value)) return fail(DCT16A_EDOMAIN, "codec path %d not built into this library", value);
        g_codec_path.store(value);
        return DCT16A_OK;
    }
    if (option == DCT16A_OPT_FWD_STORE) {
        if (!store_mode_built(value)) return fail(DCT16A_EDOMAIN, "forward store mode %d not built into this library", value);
        g_fwd_store.store(value);
        return DCT16A_OK;
    }
    if (option == DCT16A_OPT_UNIFORM_QUANT) {
        if (!uniform_quant_valid(value)) return fail(DCT16A_EDOMAIN, "uniform quantiser choice %d not in {0, 1, 2}", value);
        g_uniform_quant.store(value);
        return DCT16A_OK;
    }
    return fail(DCT16A_EDOMAIN, "unknown option %d", option);
}

DCT16A_API int dct16a_get_option(int option) {
    if (option != DCT16A_OPT_CODEC_PATH && option != DCT16A_OPT_FWD_STORE && option != DCT16A_OPT_UNIFORM_QUANT)
        return fail(DCT16A_EDOMAIN, "unknown option %d", option);
    return get_option(option);
}

DCT16A_API const char* dct16a_last_error(void) { return g_err; }

DCT16A_API const char* dct16a_version(void) { return "dct16a 0.2.0 sm_100a"; }

}  // extern "C"
