/*
 * dct16a.h — C ABI of the B200-native batched 16x16 approximate-DCT path of
 * arXiv 1606.05562 ("A multiplierless 16-point DCT approximation", the matrix T
 * of PAPER.md:270-287, evaluated with the 60-addition factorisation
 * T = P2·M4·M3·M2·P1·M1 of Eq. (1)).
 *
 * Every entry point is asynchronous on the given CUDA stream (`stream` is a
 * cudaStream_t passed as void*; NULL = legacy default stream).  All data
 * pointers are DEVICE pointers unless the name says `host`.  The caller owns
 * and frees every buffer; the library never allocates device memory and
 * never synchronises the stream.  Constants live in __constant__ memory; the
 * only state is the dynamic tile schedulers' counters (static __device__
 * arrays of 64 slots per kernel family, taken round-robin by successive calls
 * and reset by each launch's last warp) and, on the host, one completion event
 * per slot: a call whose slot was last used by a launch on ANOTHER stream that
 * may still be running makes its own stream wait for that launch first
 * (cudaStreamWaitEvent), so concurrent launches never share a counter, however
 * many are in flight.  A call made while its stream is being captured into a
 * CUDA graph takes no slot (static tile schedule: replays may overlap freely).
 * Calls are thread-safe and re-entrant.
 *
 * Errors: every function validates all arguments synchronously before any
 * launch and returns 0 on success or a negative DCT16A_E* code, leaving the
 * outputs untouched on a validation error.  dct16a_last_error() returns a
 * thread-local message for the last failure of the calling thread.  Device
 * faults surface at the caller's next synchronisation.
 *
 * Pixels: bit_depth 8 -> uint8 samples; bit_depth 10 -> int16 samples that
 * MUST lie in [0, 1023] (values outside give undefined coefficients: the
 * kernels use 16-bit SWAR lanes sized for that range).
 *
 * Blocks: each image is cut into disjoint 16x16 blocks A_k in row-major block
 * order (all blocks, reading A3 of DESIGN.md).  Block
 * (n, by, bx) has linear index b = (n·BY + by)·BX + bx with BY = height/16 and
 * BX = width/16.
 *
 * Coefficients: Z = T·X·Tᵀ per block (PAPER.md:870-880 with the scale S
 * absorbed into quantisation; k = row = vertical frequency,
 * reading A5), stored block-major int32: coef[b·256 + 16·k + l] (reading A17).
 * The pitch applies to the image side only.
 */
#ifndef DCT16A_H
#define DCT16A_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define DCT16A_API __attribute__((visibility("default")))
#else
#define DCT16A_API
#endif

/* ---- return codes ------------------------------------------------------ */
#define DCT16A_OK        0
#define DCT16A_ENULL    -1  /* a required pointer is NULL                         */
#define DCT16A_ESHAPE   -2  /* width/height not positive multiples of 16, batch<1,
                               valid_height outside (0, height]                   */
#define DCT16A_EPITCH   -3  /* pitch < width·elem, pitch or image stride not a
                               multiple of 16, image stride < pitch·height (batch>1) */
#define DCT16A_EALIGN   -4  /* a device pointer is not 16-byte aligned (TMA)      */
#define DCT16A_EDOMAIN  -5  /* r outside [1,256], step < 1, unknown mode,
                               bit_depth not 8 or 10, r range empty               */
#define DCT16A_ECUDA    -6  /* kernel launch, copy or tensor-map encode failed    */

/* ---- image batch descriptor -------------------------------------------- */
typedef struct dct16a_desc {
    int32_t width;          /* pixels per row, multiple of 16                     */
    int32_t height;         /* rows per image, multiple of 16                     */
    int32_t valid_height;   /* rows counted by SSE/PSNR, 0 < valid_height <= height
                               (1080 for 1088-padded frames, reading A13)         */
    int32_t batch;          /* number of images / frames                          */
    int32_t bit_depth;      /* 8 (uint8) or 10 (int16 in [0,1023])                */
    int32_t reserved;       /* must be 0                                          */
    int64_t pitch_bytes;    /* bytes between rows, multiple of 16                 */
    int64_t image_stride_bytes; /* bytes between images, multiple of 16           */
} dct16a_desc;

/* ---- quantiser parameters (S folded in) -------------- */
#define DCT16A_ZONAL    0   /* keep the first r zig-zag coefficients */
#define DCT16A_UNIFORM  1   /* q = sign(B)·floor(|B|/step + 1/2), B = Z/sqrt(g_k·g_l)
                               (reading A9; decided exactly in integers)           */
typedef struct dct16a_quant {
    int32_t mode;           /* DCT16A_ZONAL or DCT16A_UNIFORM                     */
    int32_t r;              /* zonal: retained coefficients, 1..256               */
    int32_t step;           /* uniform: integer step Δ >= 1                       */
    int32_t reserved;       /* must be 0                                          */
} dct16a_quant;

/*
 * dct16a_forward — Z = T·X·Tᵀ for every block (separable
 * row/column passes of the Eq. (1) network as in PAPER.md:1072-1090).
 *   src  : image batch laid out as described by *desc (uint8 or int16).
 *   coef : int32 output, batch·BY·BX·256 entries, block-major (see above);
 *          must not overlap src (DCT16A_EDOMAIN).
 * Integer-exact.  |Z| <= 65280 (8-bit) / 261888 (10-bit).
 * Scheduling: the kernel hands out tiles from a device-side counter (a
 * compact write window; slot rules in the file header).
 */
DCT16A_API int dct16a_forward(const void* src, const dct16a_desc* desc,
                              int32_t* coef, void* stream);

/*
 * dct16a_forward16 — the same Z = T·X·Tᵀ for 8-bit images, stored in 16 bits
 * (SURVEY.md §8(f) f4): every AC coefficient fits int16 (|Z| <= 32640) and
 * Z_00 = block sum fits uint16 ([0, 65280]).  coef16[b·256 + 16·k + l] holds the
 * low 16 bits of Z: read the DC entry (k = l = 0) as uint16 and every other
 * entry as int16.  Half the output bytes of dct16a_forward.
 * Errors: DCT16A_EDOMAIN unless bit_depth = 8.
 */
DCT16A_API int dct16a_forward16(const void* src, const dct16a_desc* desc, int16_t* coef16,
                                void* stream);

/*
 * dct16a_quantize — the quantisation stage with S folded in.
 *   coef   : int32 block-major Z as written by dct16a_forward.
 *   qcoef  : int32 out, same shape.  Zonal: Z ⊙ M_r (M_r = first r zig-zag
 *            positions, reading A4).  Uniform: the integer
 *            levels q (exact decision, ties away from zero).
 *   scaled : optional float32 out (may be NULL), same shape.  Zonal:
 *            s_k·s_l·(Z ⊙ M_r) = B′ of PAPER.md:874-894.  Uniform: s_k·s_l·Z = B.
 *            Here s = diag(S) of PAPER.md:315-329.
 */
DCT16A_API int dct16a_quantize(const int32_t* coef, const dct16a_desc* desc,
                               const dct16a_quant* quant, int32_t* qcoef,
                               float* scaled, void* stream);

/*
 * dct16a_inverse — A′ = Ĉᵀ·B′·Ĉ, rounded half away from
 * zero and clamped to [0, 2^b - 1] (reading A6), written as pixels.
 *   qcoef : int32 levels from dct16a_quantize (zonal: Z ⊙ M_r; uniform: q).
 *   recon : pixels in the layout, pitch and type of *desc.
 * Zonal reconstruction is exact: N = Tᵀ·(W ⊙ qcoef)·T with W = 2304/(g_k·g_l)
 * and pixel = round(N/2304) decided on the integer N.  Uniform reconstruction
 * evaluates Tᵀ·(Δ·q·s_k·s_l)·T in float64 (reading A10).
 */
DCT16A_API int dct16a_inverse(const int32_t* qcoef, const dct16a_desc* desc,
                              const dct16a_quant* quant, void* recon, void* stream);

/*
 * dct16a_psnr — per-image SSE over the first valid_height rows and
 * PSNR = 10·log10(peak²·P/SSE), peak = 2^b - 1, P = valid_height·width,
 * +INFINITY when SSE = 0 (readings A7/A13).
 *   ref, test : two image batches with the same *desc.
 *   sse       : uint64 out [batch] (exact).
 *   psnr      : optional float64 out [batch] (may be NULL).
 * DCT16A_ESHAPE if one image's valid region is 32 GiB or more.
 */
DCT16A_API int dct16a_psnr(const void* ref, const void* test, const dct16a_desc* desc,
                           uint64_t* sse, double* psnr, void* stream);

/*
 * dct16a_codec — the fused path forward -> quantise -> inverse -> SSE/PSNR
 * in one pass over the input.  Results are identical,
 * byte for byte, to dct16a_forward -> dct16a_quantize -> dct16a_inverse ->
 * dct16a_psnr.
 *   recon : optional pixels out (may be NULL: nothing is written), in the
 *           layout, pitch, image stride and type of *desc — one descriptor
 *           describes both src and recon; its byte range must not intersect
 *           src's (DCT16A_EDOMAIN).
 *   sse   : uint64 out [batch] (exact; overwritten, not accumulated).
 *   psnr  : optional float64 out [batch] (may be NULL).
 * Scheduling: as dct16a_forward (file header).
 */
DCT16A_API int dct16a_codec(const void* src, const dct16a_desc* desc,
                            const dct16a_quant* quant, void* recon,
                            uint64_t* sse, double* psnr, void* stream);

/*
 * dct16a_codec_allreduce — dct16a_codec with the path's only exchange fused
 * into the kernel (config 4 across GPUs):
 * instead of a local SSE vector and a separate all-reduce, every image's SSE
 * is added with system-scope 64-bit atomics into sse_peers[q][frame_offset + n]
 * for every q < n_peers — the per-frame SSE vectors of all ranks, mapped into
 * this device's address space (e.g. torch symmetric memory buffer_ptrs over
 * NVLink).  Integer adds: every rank ends with the exact sums, independent of
 * order.  The caller zeroes every rank's vector and synchronises the ranks
 * before the call, and again after every rank's kernel has completed, before
 * reading; PSNR follows from the summed vector.
 *   sse_peers   : HOST array of n_peers device pointers (each 8-byte aligned).
 *   n_peers     : 1..8.
 *   frame_offset: index of this call's first image in the global vector.
 * Runs the warp-per-block-pair kernel for every mode.  Errors as dct16a_codec;
 * DCT16A_EDOMAIN for n_peers outside [1, 8] or frame_offset < 0.
 */
DCT16A_API int dct16a_codec_allreduce(const void* src, const dct16a_desc* desc, const dct16a_quant* quant,
                                      void* recon, uint64_t* const* sse_peers, int32_t n_peers,
                                      int64_t frame_offset, void* stream);

/*
 * dct16a_codec_allreduce_multicast — dct16a_codec_allreduce through an NVLS
 * multicast address: sse_multicast maps the per-frame SSE
 * vectors of every GPU of the group (e.g. torch symmetric memory
 * multicast_ptr on an NVSwitch system); each image's SSE is added with one
 * multimem.red.relaxed.sys.global.add.u64, which the switch applies to every
 * GPU's copy.  Same ordering contract as dct16a_codec_allreduce (zero and
 * synchronise every rank before, synchronise after).  Passing an address that
 * is not a multicast mapping is undefined (the instruction faults).
 * Errors as dct16a_codec_allreduce.
 */
DCT16A_API int dct16a_codec_allreduce_multicast(const void* src, const dct16a_desc* desc, const dct16a_quant* quant,
                                                void* recon, uint64_t* sse_multicast, int64_t frame_offset,
                                                void* stream);

/*
 * dct16a_ssim — mean SSIM per image (Wang et al. 2004):
 * 11x11 Gaussian window (sigma 1.5, unit sum), K1 = 0.01, K2 = 0.03,
 * L = 2^b - 1, full resolution, averaged over every window position that lies
 * inside the first valid_height rows (reading A21).  Computed in float64;
 * independent of scheduling (fixed-point 2^-32 accumulation of tile sums).
 *   ref, test : two image batches with the same *desc.
 *   ssim      : float64 out [batch].
 * Errors: DCT16A_ESHAPE if valid_height < 11.
 */
DCT16A_API int dct16a_ssim(const void* ref, const void* test, const dct16a_desc* desc, double* ssim,
                           void* stream);

/*
 * dct16a_zonal_sweep — the zonal path of dct16a_codec for every retained
 * count r = r_first .. r_first + r_count - 1 in one pass over the images: the
 * r-sweep of the paper's compression experiment (Figs. 1-2;
 * config 5).  Since M_r adds one zig-zag cell (k, l) to M_{r-1}, the exact
 * numerator is updated by W_kl·Z_kl·T_k ⊗ T_l per step; every per-r result is
 * identical to dct16a_codec(mode = zonal, r, recon = NULL).
 *   sse  : uint64 out [batch][r_count]; sse[n·r_count + i] is the SSE of image
 *          n over its valid rows reconstructed with r = r_first + i.
 *   psnr : optional float64 out, same layout (+INFINITY where SSE = 0).
 * Errors: DCT16A_EDOMAIN unless 1 <= r_first and r_first + r_count - 1 <= 256
 * with r_count >= 1.  Work grows with r_first + r_count (the sweep starts at 1).
 */
DCT16A_API int dct16a_zonal_sweep(const void* src, const dct16a_desc* desc, int32_t r_first,
                                  int32_t r_count, uint64_t* sse, double* psnr, void* stream);

/*
 * dct16a_sse_psnr — the PSNR finaliser of the path (PAPER.md:906-910,
 * readings A7/A8) on its own: for `count` per-image SSE values of images
 * described by *desc (peak 2^b - 1, P = valid_height·width pixels each;
 * desc->batch is not used), writes
 *   psnr[i]     = 10·log10(peak²·P/sse[i]), +INFINITY for 0     (may be NULL),
 *   *sse_total  = Σ sse[i], exact                              (may be NULL),
 *   *psnr_total = 10·log10(peak²·P·count/Σ sse[i])             (may be NULL):
 * config 4's global PSNR over all frames after the SSE all-reduce.
 *   sse : DEVICE uint64 [count]; outputs are DEVICE pointers, 8-byte aligned.
 * Errors: DCT16A_ESHAPE for count outside [1, 2^31).
 */
DCT16A_API int dct16a_sse_psnr(const uint64_t* sse, int64_t count, const dct16a_desc* desc, double* psnr,
                               uint64_t* sse_total, double* psnr_total, void* stream);

/*
 * dct16a_forward_host — dct16a_forward end to end from HOST memory: the
 * images are read from host_src (laid out as *desc describes) and Z is
 * written to host_coef (int32, block-major, batch·BY·BX·256 entries).  The
 * batch is cut into chunks of whole images; chunk i is copied host->device
 * (one cudaMemcpyAsync), transformed, and copied device->host (one
 * cudaMemcpyAsync) on the i-th of two library-owned streams (created once per
 * device, joined to `stream` by events), so copies in both directions overlap
 * each other and the transform.  Asynchronous on `stream` like every entry:
 * synchronise it before reading host_coef.  host_src / host_coef should be
 * page-locked (cudaHostAlloc / pinned torch tensors) for the copies to overlap.
 *   workspace       : DEVICE scratch, 1024-byte aligned, owned by the caller,
 *                     holding two chunk slots (input + coefficients);
 *   workspace_bytes : its size; the chunk is the largest number of images
 *                     whose two slots fit.
 * Errors: DCT16A_EDOMAIN if the workspace holds less than one image per slot
 * (see dct16a_forward_host_workspace); DCT16A_EALIGN for a misaligned workspace.
 */
DCT16A_API int dct16a_forward_host(const void* host_src, const dct16a_desc* desc, int32_t* host_coef,
                                   void* workspace, int64_t workspace_bytes, void* stream);

/* Workspace bytes dct16a_forward_host needs for chunks of `chunk_images`
 * images (negative DCT16A_E* code on a bad descriptor or chunk_images < 1). */
DCT16A_API int64_t dct16a_forward_host_workspace(const dct16a_desc* desc, int32_t chunk_images);

/*
 * dct16a_set_option / dct16a_get_option — process-wide knobs for tuning and
 * cross-checking; they never change results (every kernel choice computes the
 * same bytes).  Initial values come from the environment variables named
 * below; set_option returns DCT16A_EDOMAIN for an unknown option or value.
 *   DCT16A_OPT_CODEC_PATH (env DCT16A_CODEC_PATH): fused-codec kernel choice,
 *     0 = automatic (default): every zonal case on the band-pruned
 *         warp-per-tile kernel (8- and 10-bit, any r), uniform on the
 *         warp-per-block-pair kernel;
 *     2 = always the warp-per-block-pair kernel.
 *     (Libraries built with -DDCT16A_EXPERIMENTS also take 1 = zonal on the
 *     generic kernel and 3 = zonal 8-bit r <= 36 on the thread-per-block kernel.)
 *   DCT16A_OPT_FWD_STORE (env DCT16A_FWD_STORE): output path of the forward
 *     kernel, -1 = default (5 for 8-bit, 3 for 10-bit), 3 = 8 KB TMA stores,
 *     5 = one 32 KB TMA store per tile (experiment builds: 0..7, the variants
 *     of profiles/r01_fwd_store_modes.md).
 *   DCT16A_OPT_UNIFORM_QUANT (env DCT16A_UNIFORM_QUANT): the fused codec's
 *     uniform quantiser (reading A9; both decide every level exactly),
 *     0 = automatic (default): 64-bit fixed point for steps <= 8, float32 above;
 *     1 = always float32; 2 = fixed point wherever its error bound allows it
 *     (steps up to ~170 for 10-bit, ~680 for 8-bit input), float32 beyond.
 * A value the library was not built with returns DCT16A_EDOMAIN (from the
 * environment it is ignored).
 */
#define DCT16A_OPT_CODEC_PATH    1
#define DCT16A_OPT_FWD_STORE     2
#define DCT16A_OPT_UNIFORM_QUANT 3
DCT16A_API int dct16a_set_option(int option, int value);
DCT16A_API int dct16a_get_option(int option);

/* Thread-local description of the calling thread's last failure ("" if none). */
DCT16A_API const char* dct16a_last_error(void);

/* Library version and build target, e.g. "dct16a 0.2.0 sm_100a". */
DCT16A_API const char* dct16a_version(void);

#ifdef __cplusplus
}
#endif
#endif /* DCT16A_H */
