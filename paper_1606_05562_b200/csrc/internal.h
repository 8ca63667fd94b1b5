// internal.h — private launcher interface between the C-ABI layer (abi.cu)
// and the kernel translation units.  Not installed; not part of the ABI.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/dct16a.h"

namespace dct16a {

// Geometry of a validated image batch, in blocks.
struct Geom {
    int W, H, VH, N, bits;   // width, height, valid height, batch, bit depth
    int BX, BY;              // blocks per row / column
    int elem;                // bytes per pixel (1 or 2)
    int64_t pitch, istride;  // bytes
    int64_t nblocks;         // N·BY·BX
};

// Encodes a tiled tensor map through the driver entry point (no -lcuda link).
// Returns 0 on success, a CUresult otherwise.
int encode_tiled(CUtensorMap* map, CUtensorMapDataType dt, uint32_t rank, const void* gaddr,
                 const uint64_t* dims, const uint64_t* strides_bytes, const uint32_t* box,
                 CUtensorMapSwizzle swz, CUtensorMapL2promotion promo);

int num_sms();

// Opt a kernel into `bytes` of dynamic shared memory on the current device, once
// per (kernel, device): the attribute is per device, so a process driving
// several GPUs must set it on each.  Returns a cudaError_t.
int smem_optin(const void* func, int bytes);

// Launchers: return cudaError_t of the launch (cudaSuccess = 0) or a negative
// DCT16A_E* code for encode failures.
int launch_forward(const void* src, const Geom& g, int32_t* coef, cudaStream_t st);
int launch_forward16(const void* src, const Geom& g, int16_t* coef, cudaStream_t st);
int launch_quantize(const int32_t* coef, const Geom& g, const dct16a_quant& q, int32_t* qcoef,
                    float* scaled, cudaStream_t st);
int launch_inverse(const int32_t* qcoef, const Geom& g, const dct16a_quant& q, void* recon,
                   cudaStream_t st);
int launch_psnr(const void* ref, const void* test, const Geom& g, uint64_t* sse, double* psnr,
                cudaStream_t st);
int launch_codec(const void* src, const Geom& g, const dct16a_quant& q, void* recon,
                 uint64_t* sse, double* psnr, cudaStream_t st);
// Smallest anti-diagonal band k + l <= d holding the first r zig-zag positions.
int zonal_band(int r);
// Whether the band-pruned zonal kernel (zonal_band.cu) covers a case.
bool zonal_band_applies(const Geom& g, int r);
int launch_zonal_band(const void* src, const Geom& g, int r, void* recon, uint64_t* sse, cudaStream_t st);
#ifdef DCT16A_EXPERIMENTS
// thread-per-block zonal codec (codec path 3), same applicability as the band kernel
int launch_zonal_tpb(const void* src, const Geom& g, int r, void* recon, uint64_t* sse, cudaStream_t st);
#endif
// warp-per-block-pair codec (uniform, and zonal cases zonal_tpb does not take)
int launch_codec_warp(const void* src, const Geom& g, const dct16a_quant& q, void* recon, uint64_t* sse,
                      cudaStream_t st);
#ifdef DCT16A_EXPERIMENTS
// uniform-quantiser codec, two blocks per lane (codec_uniform.cu); n_peers = 0: local sse
int launch_codec_uniform(const void* src, const Geom& g, const dct16a_quant& q, void* recon, uint64_t* sse,
                         cudaStream_t st, uint64_t* const* peers, int n_peers, long long frame_offset, int multicast);
#endif
// mean SSIM per image (ssim.cu)
int launch_ssim(const void* ref, const void* test, const Geom& g, double* ssim, cudaStream_t st);
// zonal r-sweep (sweep.cu) and the shared PSNR finaliser
int launch_sweep(const void* src, const Geom& g, int r_first, int r_count, uint64_t* sse, double* psnr,
                 cudaStream_t st);
int launch_psnr_finish(const Geom& g, long long count, uint64_t* sse, double* psnr, cudaStream_t st);
// exact sum of `count` SSE values and the PSNR of the whole set (P·count pixels)
int launch_sse_total(const Geom& g, long long count, const uint64_t* sse, uint64_t* total, double* psnr_total,
                     cudaStream_t st);
// fused codec + SSE all-reduce over peer memory (codec_warp.cu)
int launch_codec_allreduce(const void* src, const Geom& g, const dct16a_quant& q, void* recon,
                           uint64_t* const* peers, int n_peers, long long frame_offset, int multicast,
                           cudaStream_t st);
// library options (dct16a_set_option); read by the launchers
int get_option(int option);

// Host side of the tile schedulers (sched.cuh).  A launcher holds one guard
// around its kernel launch: the guard gives the launch a counter slot of its
// kernel family that no unfinished launch on another stream still uses (it
// makes `st` wait on the slot's previous launch when that one may still be
// running), records the slot's completion event after the launch and keeps the
// family's slot table locked in between.  A launch being captured into a CUDA
// graph gets slot -1: the static schedule, so overlapping replays of one graph
// are safe.
enum SchedFamily { kSchedForward = 0, kSchedBand = 1, kSchedCodecWarp = 2, kSchedCodecUniform = 3, kSchedFamilies = 4 };
class SchedGuard {
  public:
    SchedGuard(int family, cudaStream_t st);
    ~SchedGuard();
    SchedGuard(const SchedGuard&) = delete;
    SchedGuard& operator=(const SchedGuard&) = delete;
    int slot() const { return slot_; }   // -1: static schedule
    int error() const { return err_; }   // cudaError_t of the slot hand-over (0 = fine)

  private:
    void* state_ = nullptr;
    cudaStream_t st_;
    int slot_ = -1, err_ = 0;
};

}  // namespace dct16a
