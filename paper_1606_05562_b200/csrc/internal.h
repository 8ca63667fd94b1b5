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
// thread-per-block zonal codec for 8-bit and small bands; returns 1 if not applicable
int launch_zonal_tpb(const void* src, const Geom& g, int r, void* recon, uint64_t* sse, cudaStream_t st);
int launch_zonal_band(const void* src, const Geom& g, int r, void* recon, uint64_t* sse, cudaStream_t st);
int zonal_band(int r);
// warp-per-block-pair codec (uniform, and zonal cases zonal_tpb does not take)
int launch_codec_warp(const void* src, const Geom& g, const dct16a_quant& q, void* recon, uint64_t* sse,
                      cudaStream_t st);
// mean SSIM per image (ssim.cu)
int launch_ssim(const void* ref, const void* test, const Geom& g, double* ssim, cudaStream_t st);
// zonal r-sweep (sweep.cu) and the shared PSNR finaliser
int launch_sweep(const void* src, const Geom& g, int r_first, int r_count, uint64_t* sse, double* psnr,
                 cudaStream_t st);
int launch_psnr_finish(const Geom& g, long long count, uint64_t* sse, double* psnr, cudaStream_t st);
// fused codec + SSE all-reduce over peer memory (codec_warp.cu)
int launch_codec_allreduce(const void* src, const Geom& g, const dct16a_quant& q, void* recon,
                           uint64_t* const* peers, int n_peers, long long frame_offset, cudaStream_t st);
// library options (dct16a_set_option); read by the launchers
int get_option(int option);

}  // namespace dct16a
