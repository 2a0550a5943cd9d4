/*
 * kmd.h -- C ABI of libkmd: the B200 (sm_100a) kernel-map decoder, per-pixel
 * filter and kernel fusion of arXiv 2202.05977 ("weight sharing kernel
 * prediction"), reconstruction phase.
 *
 * What one call computes (§3 Eq. 3-5, §4.2, §5.3), for every frame n
 * and pixel p, with M importance maps I_i and kernel sizes k_i:
 *
 *   w_p^i(q) = exp(I_i(q)) / sum_{q' in Omega_{k_i}(p)} exp(I_i(q'))  (Eq. 3)
 *   R^{k_i}(p,c) = sum_{q in Omega_{k_i}(p)} w_p^i(q) r_c(q)          (Eq. 4)
 *   alpha_i(p)   = softmax_i(B_i(p))
 *   Rhat(p,c)    = sum_i alpha_i(p) R^{k_i}(p,c)                       (Eq. 5)
 *
 * Omega_k(p) is the k x k window centred on p; samples outside the image are
 * clamped to the nearest edge pixel, for the importance unfold and for the
 * colour taps alike (reading R1).  The H x W x k^2 kernel map of
 * Fig. 3 is never written to memory: one streaming kernel builds, applies and
 * fuses the kernels ("one single function ... in a
 * streaming manner").
 *
 * Conventions for every entry point
 *  - Types: fp32 in, fp32 out, fp32 arithmetic.  Planar, row-major,
 *    contiguous ("NCHW"):  radiance [N,3,H,W]  importance [N,M,H,W]
 *    blend [N,M,H,W]  out [N,3,H,W].
 *  - Memory: device pointers unless the name ends in _host.  The caller owns
 *    every buffer; the library allocates nothing per call and keeps no mutable
 *    global state except a thread-local error string (reentrant).
 *  - Asynchrony: argument checks run synchronously, before any CUDA call;
 *    work is enqueued on `stream` (a cudaStream_t; NULL = legacy default
 *    stream) and the call returns without synchronising.
 *  - Errors: returned as kmd_status; nothing is thrown or aborted across the
 *    ABI.  kmd_last_error() gives a human-readable detail for this thread.
 *  - Aliasing: `out` must not overlap any input (the stencil reads
 *    neighbours) -> KMD_ERR_ALIAS.
 *  - Numerics: max relative error <= 1e-5 against the fp64 oracle for finite
 *    inputs with radiance >= 0.  Every kernel evaluates Eq. 3
 *    with unshifted exp(I) (any shift cancels, reading R2) and guards the
 *    range as follows (reading R13):
 *      TMA kernel (W % 4 == 0, 16-B aligned, k <= 13; kmd_last_kernel() 3,
 *      100+M, 150+M, 200+M): per output PIXEL.  A pixel is recomputed by a
 *      per-window max-shifted evaluation (IEEE expf and division) when, for
 *      any size, its box denominator sum_q exp(I(q)) lies outside
 *      [1e-30, 1e30] (this includes overflow to +inf), when the sum of its
 *      fusion weights exp(B_i) lies outside [1e-30, 1e30], or when its result
 *      is not finite.
 *      Other kernels (kmd_last_kernel() 1, 2): per (tile, size).  A tile whose
 *      importance values leave [KMD_EXP_SAFE_LO, KMD_EXP_SAFE_HI] or whose
 *      |radiance| exceeds KMD_RADIANCE_SAFE takes the max-shifted path.
 *    Either way the result is the same operation; only the speed differs.
 */
#ifndef KMD_H
#define KMD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KMD_VERSION_MAJOR 0
#define KMD_VERSION_MINOR 1

#define KMD_MAX_SIZES 8        /* M <= 8 maps per call (the paper uses 6) */
#define KMD_MAX_K 31           /* largest odd window size accepted                      */
#define KMD_EXP_SAFE_LO (-60.0f)
#define KMD_EXP_SAFE_HI (60.0f)
#define KMD_RADIANCE_SAFE (1.0e8f)

typedef enum {
    KMD_OK = 0,
    KMD_ERR_NULL = 1,   /* a required pointer is NULL (blend may be NULL only when M == 1)  */
    KMD_ERR_CONFIG = 2, /* M not in [1,8]; a size even, < 1, > KMD_MAX_K or > min(H,W);
                           border not KMD_BORDER_CLAMP                                       */
    KMD_ERR_DIM = 3,    /* N < 0, H < 1 or W < 1 (when N > 0); bad band geometry;
                           element count overflows int64                                      */
    KMD_ERR_ALIGN = 4,  /* kmd_decode_filter_fuse_bf16 only: W % 8 != 0 or a buffer not
                           16-byte aligned (the fp32 entry points accept any 4-byte pointer)  */
    KMD_ERR_ALIAS = 5,  /* out overlaps an input                                              */
    KMD_ERR_CUDA = 6,   /* a CUDA runtime call or launch failed (see kmd_last_error)          */
    KMD_ERR_NCCL = 7    /* NCCL unavailable or an NCCL call failed (kmd_halo_exchange etc.) */
} kmd_status;

typedef enum { KMD_BORDER_CLAMP = 0 } kmd_border;

/* Kernel-size set and fusion options (SPEC.md:228-231 FusionConfig). */
typedef struct {
    int32_t num_sizes;              /* M, 1..KMD_MAX_SIZES                                  */
    int32_t sizes[KMD_MAX_SIZES];   /* odd window sizes; importance map i <-> sizes[i]
                                       (paper: {3,5,7,9,11,13} = k_b + i*k_s, k_b=3, k_s=2)  */
    int32_t blend_is_logits;        /* 1: blend holds logits, softmax applied inside (paper,
                                       PAPER.md:251); 0: blend already holds alpha_i(p)      */
    int32_t border;                 /* KMD_BORDER_CLAMP (the only policy, R1)     */
} kmd_config;

typedef void* kmd_stream_t;         /* a cudaStream_t */

/* ---------------------------------------------------------------------------
 * Hot path: fused decode (Eq. 3) + filter (Eq. 4) + fusion (Eq. 5).
 *   radiance   [N,3,H,W] device, noisy demodulated HDR irradiance
 *   importance [N,M,H,W] device, importance maps I_i (Eq. 2; map i <-> cfg->sizes[i])
 *   blend      [N,M,H,W] device, fusion logits (or alphas); NULL allowed iff M == 1
 *   out        [N,3,H,W] device, the fused result Rhat
 * N == 0 is a no-op.  Errors: NULL, CONFIG, DIM, ALIAS, CUDA.                 */
kmd_status kmd_decode_filter_fuse(const float* radiance, const float* importance,
                                  const float* blend, float* out, int32_t N, int32_t H,
                                  int32_t W, const kmd_config* cfg, kmd_stream_t stream);

/* Hot path with bf16 importance maps and fusion logits (NEXT row 4's
 * alternative: the network's output in low precision; the
 * radiance and the result stay fp32 since the paper's path filters HDR
 * irradiance).  Same operation as kmd_decode_filter_fuse on the
 * bf16 values widened exactly to fp32 (R24).
 *   importance [N,M,H,W] device, bf16 bit patterns (e.g. torch.bfloat16 storage)
 *   blend      [N,M,H,W] device, bf16; NULL allowed iff M == 1
 *   radiance, out as kmd_decode_filter_fuse (fp32)
 * Runs on the TMA kernel only: needs W % 8 == 0 and 16-byte aligned buffers
 * (else KMD_ERR_ALIGN) and every size <= 13 (else KMD_ERR_CONFIG).
 * Other errors as kmd_decode_filter_fuse.                                     */
kmd_status kmd_decode_filter_fuse_bf16(const float* radiance, const uint16_t* importance,
                                       const uint16_t* blend, float* out, int32_t N, int32_t H,
                                       int32_t W, const kmd_config* cfg, kmd_stream_t stream);

/* Hot path + remodulation epilogue (NEXT row 1; Fig. 1, 258: "we
 * filter the noisy input irradiance without albedo, and at the last step, we
 * multiply back the albedo"): out = Rhat * albedo, in the same pass.
 *   albedo [N,3,H,W] device (NULL = plain kmd_decode_filter_fuse); other
 *   arguments, errors and numerics as kmd_decode_filter_fuse.               */
kmd_status kmd_decode_filter_fuse_remod(const float* radiance, const float* importance,
                                        const float* blend, const float* albedo, float* out,
                                        int32_t N, int32_t H, int32_t W, const kmd_config* cfg,
                                        kmd_stream_t stream);

/* Albedo demodulation before filtering:
 * irradiance = radiance / max(albedo, eps), elementwise over [N,3,H,W] device
 * buffers; eps > 0 (else KMD_ERR_CONFIG); irradiance may alias radiance.     */
kmd_status kmd_demodulate(const float* radiance, const float* albedo, float eps, float* irradiance,
                          int32_t N, int32_t H, int32_t W, kmd_stream_t stream);

/* Remodulation on its own: out = irradiance * albedo. */
kmd_status kmd_remodulate(const float* irradiance, const float* albedo, float* out, int32_t N,
                          int32_t H, int32_t W, kmd_stream_t stream);

/* One size, no fusion: out_i = R^{k}(p,c) of Eq. 3-4.
 *   radiance [N,3,H,W], importance_i [N,1,H,W], out_i [N,3,H,W], all device.   */
kmd_status kmd_decode_filter(const float* radiance, const float* importance_i, float* out_i,
                             int32_t N, int32_t H, int32_t W, int32_t k,
                             kmd_stream_t stream);

/* Fusion only (Eq. 5):
 *   filtered [N,M,3,H,W] device (R^{k_i}), blend [N,M,H,W] device (NULL iff M == 1),
 *   out [N,3,H,W] device.                                                       */
kmd_status kmd_fuse(const float* filtered, const float* blend, float* out, int32_t N,
                    int32_t H, int32_t W, int32_t M, int32_t blend_is_logits,
                    kmd_stream_t stream);

/* Row band of a taller frame (multi-GPU spatial split).
 * The frame has H_global rows; this call produces output rows
 * [y0, y0 + band_rows).  radiance / importance hold rows
 * [y0 - halo_top, y0 + band_rows + halo_bot) of the frame:
 *   radiance [N,3,halo_top+band_rows+halo_bot,W], importance [N,M,...,W];
 * blend and out hold only the band: [N,M,band_rows,W] and [N,3,band_rows,W].
 * Rows outside the frame are clamped to rows 0 / H_global-1 as in the whole-
 * frame call, so the band outputs are bitwise equal to the corresponding rows
 * of kmd_decode_filter_fuse on the whole frame.  Requires
 *   halo_top >= min(r_max, y0) and halo_bot >= min(r_max, H_global - y0 - band_rows),
 * r_max = (max_i k_i - 1)/2, and y0 - halo_top >= 0,
 * y0 + band_rows + halo_bot <= H_global.  Errors as kmd_decode_filter_fuse.  */
kmd_status kmd_decode_filter_fuse_band(const float* radiance, const float* importance,
                                       const float* blend, float* out, int32_t N,
                                       int32_t band_rows, int32_t W, int32_t halo_top,
                                       int32_t halo_bot, int32_t y0, int32_t H_global,
                                       const kmd_config* cfg, kmd_stream_t stream);

/* The band call in two parts, so the halo exchange can overlap the work that
 * does not need it.  part = KMD_BAND_ALL: the whole band
 * (== kmd_decode_filter_fuse_band).  KMD_BAND_INTERIOR: only the output rows
 * whose windows read owned rows alone (rows [y0, y0 + band_rows), plus frame
 * edges clamped where halo_top / halo_bot is 0); the halo rows of radiance and
 * importance are not read and may be in flight.  KMD_BAND_SEAMS: every other
 * output row of the band (the rows next to a non-empty halo).  INTERIOR then
 * SEAMS write every output row exactly once, bitwise equal to KMD_BAND_ALL.
 * The split follows the TMA kernel's global tile grid; when
 * another kernel serves the band (W % 4 != 0, unaligned, k > 13), INTERIOR
 * does nothing and SEAMS does the whole band.  Arguments and errors as
 * kmd_decode_filter_fuse_band; part outside these values -> KMD_ERR_CONFIG. */
#define KMD_BAND_ALL 0
#define KMD_BAND_INTERIOR 1
#define KMD_BAND_SEAMS 2
kmd_status kmd_decode_filter_fuse_band_part(const float* radiance, const float* importance,
                                            const float* blend, float* out, int32_t N,
                                            int32_t band_rows, int32_t W, int32_t halo_top,
                                            int32_t halo_bot, int32_t y0, int32_t H_global,
                                            const kmd_config* cfg, int32_t part, kmd_stream_t stream);

/* ---------------------------------------------------------------------------
 * Multi-GPU row bands over NCCL (configs[3]): one process per
 * GPU, one communicator over the ranks that share a frame.  libkmd loads NCCL
 * at run time (dlopen "libnccl.so.2"; in a process that imported torch this is
 * torch's NCCL); without it these calls return KMD_ERR_NCCL and nothing else
 * in the library is affected.
 *
 * kmd_nccl_unique_id: rank 0 creates the 128-byte id (NCCL_UNIQUE_ID_BYTES),
 *   which the caller broadcasts to every rank (e.g. torch.distributed).
 * kmd_comm_init: collective over nranks processes (blocking); *comm receives an
 *   opaque handle (an ncclComm_t) owned by the caller until kmd_comm_destroy.  */
#define KMD_NCCL_ID_BYTES 128
kmd_status kmd_nccl_unique_id(uint8_t id[KMD_NCCL_ID_BYTES]);
kmd_status kmd_comm_init(void** comm, const uint8_t id[KMD_NCCL_ID_BYTES], int32_t nranks, int32_t rank);
kmd_status kmd_comm_destroy(void* comm);

/* Halo exchange of one row band: ONE grouped NCCL step (ncclGroupStart /
 * ncclGroupEnd) over every plane, posted directly on the halo and edge rows
 * (each a contiguous [rows][W] block of its plane; no staging copies).
 *   planes[p]   host array of n_planes device pointers; plane p is fp32
 *               [halo_top + band_rows + halo_bot][W], owned rows filled
 *   halo        rows exchanged with each neighbour (r_max of the band call)
 *   peer_up     rank owning the rows above (its last rows are our top halo), or -1
 *   peer_down   rank owning the rows below, or -1
 *   halo_top = peer_up >= 0 ? halo : 0, halo_bot = peer_down >= 0 ? halo : 0.
 * Per plane, in this order: recv rows [0, halo_top) from peer_up; recv rows
 * [halo_top + band_rows, + halo_bot) from peer_down; send rows
 * [halo_top, halo_top + halo) to peer_up; send rows
 * [halo_top + band_rows - halo, halo_top + band_rows) to peer_down.  NCCL
 * matches the messages of one pair of ranks in posting order, so a rank that
 * is its own neighbour (peer == its rank) receives its first owned rows into
 * its top halo and its last owned rows into its bottom halo.
 * Enqueued on stream; band_rows >= halo >= 0 (else KMD_ERR_DIM); NCCL failures
 * -> KMD_ERR_NCCL.                                                            */
kmd_status kmd_halo_exchange(void* comm, float* const* planes, int32_t n_planes, int32_t band_rows,
                             int32_t W, int32_t halo, int32_t peer_up, int32_t peer_down,
                             kmd_stream_t stream);

/* One band step with the exchange overlapped: the exchange
 * of the 3 radiance and M importance planes of every frame runs on
 * comm_stream while the band interior (KMD_BAND_INTERIOR) runs on stream; the
 * seams (KMD_BAND_SEAMS) follow once the exchange is complete.  Buffers as
 * kmd_decode_filter_fuse_band with halo_top / halo_bot derived from halo and
 * the peers as in kmd_halo_exchange (radiance and importance are written:
 * their halo rows).  comm_stream == stream (or NULL) serialises the exchange
 * before the interior.  comm may be NULL when both peers are -1.  All work is
 * ordered after what was queued on stream and before what is queued on it
 * afterwards.                                                                */
kmd_status kmd_band_step(void* comm, float* radiance, float* importance, const float* blend, float* out,
                         int32_t N, int32_t band_rows, int32_t W, int32_t halo, int32_t peer_up,
                         int32_t peer_down, int32_t y0, int32_t H_global, const kmd_config* cfg,
                         kmd_stream_t stream, kmd_stream_t comm_stream);

/* End-to-end from HOST memory: copies the inputs host->device, runs the fused
 * kernel and copies the result device->host, all on `stream` (pinned host
 * buffers make the copies asynchronous and overlappable).  The caller passes a
 * device workspace of at least kmd_host_workspace_bytes(N,H,W,cfg) bytes; the
 * work is pipelined in frame chunks across the copy engines.  The call returns
 * after enqueueing; synchronise `stream` before reading out_host.  Ordering:
 * the kernels and device->host copies follow the work already queued on
 * `stream`, and `stream` resumes after the last copy; the host->device copies
 * (host inputs into the workspace) wait only until the workspace is free, so
 * consecutive calls on one host thread stream their copies back to back.
 * The workspace belongs to the library from the call until `stream` has
 * passed it; the caller must not use it for other work in between.          */
size_t kmd_host_workspace_bytes(int32_t N, int32_t H, int32_t W, const kmd_config* cfg);
kmd_status kmd_decode_filter_fuse_host(const float* radiance_host, const float* importance_host,
                                       const float* blend_host, float* out_host, int32_t N,
                                       int32_t H, int32_t W, const kmd_config* cfg,
                                       void* device_workspace, size_t workspace_bytes,
                                       kmd_stream_t stream);
/* The same with bf16 importance maps and fusion logits in host memory (the
 * network's output at 2 B per value: 75 instead of 124 MB of host->device
 * copies per 1080p M = 6 frame); the kernel is kmd_decode_filter_fuse_bf16's
 * (bf16 widened exactly to fp32, R24), run per band.  Needs W % 8
 * == 0 and sizes <= 13 (else KMD_ERR_ALIGN / KMD_ERR_CONFIG); the workspace
 * size is kmd_host_workspace_bytes(...) as above.                           */
kmd_status kmd_decode_filter_fuse_host_bf16(const float* radiance_host, const uint16_t* importance_host,
                                            const uint16_t* blend_host, float* out_host, int32_t N,
                                            int32_t H, int32_t W, const kmd_config* cfg,
                                            void* device_workspace, size_t workspace_bytes,
                                            kmd_stream_t stream);

/* ---------------------------------------------------------------------------
 * NEXT row 2: the multi-resolution "Ours MR" reconstruction (PAPER.md:313-318
 * §5.2, Eq. 7; 324 "two filtering kernels with sizes 3 and 5 for each
 * resolution"; Table 3).  Level 0 is the input resolution; level
 * l filters r_l = D^l(r_0) (D = 2x2 mean) with its own
 * importance maps and fusion logits (Eq. 3-5), then the levels are combined
 * from the coarsest:  c_{L-1} = f_{L-1},
 *   c_l = f_l - alpha_l * U D f_l + alpha_l * U c_{l+1}     (Eq. 7)
 * with U = nearest upsampling.  H and W must be divisible by
 * 2^(levels-1) (else KMD_ERR_DIM).
 *   radiance      [N,3,H,W]                      level-0 irradiance
 *   importance[l] [N,M_l,H>>l,W>>l]              per level (array of device pointers)
 *   blend[l]      [N,M_l,H>>l,W>>l] or NULL iff M_l == 1
 *   alpha[l]      [N,1,H>>l,W>>l], l < levels-1  Eq. 7 blending weight in [0,1]
 *   out           [N,3,H,W]
 *   workspace     device scratch of kmd_mr_workspace_bytes(...) bytes
 * The coarse levels run on a library-owned auxiliary stream (thread-local,
 * created on first use) forked from and joined back into `stream`, so the
 * call stays ordered on `stream` (and capturable into a CUDA graph).        */
#define KMD_MR_MAX_LEVELS 4
typedef struct {
    int32_t levels;                          /* 1..KMD_MR_MAX_LEVELS (paper: 3) */
    kmd_config level[KMD_MR_MAX_LEVELS];     /* sizes per level (paper: {3,5})  */
} kmd_mr_config;
size_t kmd_mr_workspace_bytes(int32_t N, int32_t H, int32_t W, const kmd_mr_config* cfg);
kmd_status kmd_mr_decode_filter_fuse(const float* radiance, const float* const* importance,
                                     const float* const* blend, const float* const* alpha,
                                     float* out, int32_t N, int32_t H, int32_t W,
                                     const kmd_mr_config* cfg, void* workspace,
                                     size_t workspace_bytes, kmd_stream_t stream);
/* The two MR building blocks on their own: D on [N,C,H,W] ->
 * [N,C,H/2,W/2] (H, W even), and Eq. 7 for one pair of levels:
 * fine [N,3,H,W], coarse [N,3,H/2,W/2], alpha [N,1,H,W] -> out [N,3,H,W].   */
kmd_status kmd_downsample2x2(const float* in, float* out, int32_t N, int32_t C, int32_t H,
                             int32_t W, kmd_stream_t stream);
kmd_status kmd_combine_resolutions(const float* fine, const float* coarse, const float* alpha,
                                   float* out, int32_t N, int32_t H, int32_t W,
                                   kmd_stream_t stream);

/* ---------------------------------------------------------------------------
 * NEXT row 3: backward of kmd_decode_filter_fuse w.r.t. the importance maps
 * and the fusion logits (end-to-end training, Eq. 1;
 * SPEC.md:289-297).  Given grad_out = dL/dRhat [N,3,H,W] (device):
 *   grad_importance [N,M,H,W] = dL/dI_i,  grad_blend [N,M,H,W] = dL/dB_i
 *   (dL/dalpha_i when blend_is_logits == 0; may be NULL; zeros when M == 1).
 * The radiance gradient is not computed (rendered data).
 * Every size must be <= 13 (else KMD_ERR_CONFIG).  Importance must lie in
 * (-80, 80): the backward evaluates exp(I) unshifted and has no exact
 * fallback, so values outside give inf / NaN gradients.  With a device workspace
 * of kmd_backward_workspace_bytes(...) bytes (8 M + 4 B per pixel: the
 * per-size pair s_i = a_i / den_i, d_i = G.R_i, and log sum_i exp(B_i)), W % 4 == 0 and 16-byte aligned buffers
 * (grad_importance included) the
 * TMA passes run (kmd_last_kernel() == 11); otherwise (or with workspace ==
 * NULL) a one-launch tiled kernel that needs no workspace (== 10).          */
size_t kmd_backward_workspace_bytes(int32_t N, int32_t H, int32_t W, const kmd_config* cfg);
kmd_status kmd_decode_filter_fuse_backward(const float* radiance, const float* importance,
                                           const float* blend, const float* grad_out,
                                           float* grad_importance, float* grad_blend, int32_t N,
                                           int32_t H, int32_t W, const kmd_config* cfg,
                                           void* workspace, size_t workspace_bytes,
                                           kmd_stream_t stream);

/* ---------------------------------------------------------------------------
 * NEXT row 4: the temporal accumulation pre-pass (§4.1;
 * SPEC.md:147-175), fused into one pass over [N,H,W] pixels:
 *   reproject    s = nearest pixel of p + motion(p): fx = floorf(((float)x + mx) + 0.5f),
 *                likewise fy (reading R21); in bounds iff s lies in the frame
 *                and prev_valid(s) != 0;
 *   consistency  fp32, this exact order, no FMA contraction (reading R22):
 *                d = cur_position(p) - prev_position(s),
 *                (d0*d0 + d1*d1) + d2*d2 < pos_tol*pos_tol, and with a = 2 cur_normal(p) - 1,
 *                b = 2 prev_normal(s) - 1 (normals stored in [0,1]):
 *                (a0*b0 + a1*b1) + a2*b2 > normal_tol * sqrtf(((a.a) * (b.b)));
 *   accumulate   accum = mask ? (1 - alpha) prev_radiance(s) + alpha cur_radiance(p)
 *                             : cur_radiance(p)   ("failed pixels remain original 1 spp").
 * Device buffers: radiance / position / normal [N,3,H,W] float, motion
 * [N,2,H,W] float (pixels; channel 0 = x), prev_valid [N,H,W] uint8, accum
 * [N,3,H,W] float, mask [N,H,W] uint8 or NULL.  accum may alias cur_radiance;
 * it must not overlap any prev_* buffer (KMD_ERR_ALIAS).  pos_tol > 0,
 * normal_tol in (0, 1], alpha in (0, 1], else KMD_ERR_CONFIG.               */
kmd_status kmd_temporal_accumulate(const float* cur_radiance, const float* prev_radiance,
                                   const float* prev_position, const float* prev_normal,
                                   const uint8_t* prev_valid, const float* cur_position,
                                   const float* cur_normal, const float* motion, float* accum,
                                   uint8_t* mask, int32_t N, int32_t H, int32_t W, float pos_tol,
                                   float normal_tol, float alpha, kmd_stream_t stream);

/* Algorithmic HBM bytes of one kmd_decode_filter_fuse call:
 * N*H*W*4*(3 + M + (blend? M : 0) + 3)  (inputs read once, output written once). */
int64_t kmd_algorithmic_bytes(int32_t N, int32_t H, int32_t W, const kmd_config* cfg,
                              int32_t has_blend);

/* Number of kernel launches one kmd_decode_filter_fuse call enqueues (for the
 * bench's gpu_launches count). */
int32_t kmd_launches_per_call(void);

const char* kmd_status_string(kmd_status s);
const char* kmd_last_error(void);     /* thread-local detail of the last failure */
int32_t kmd_version(void);             /* KMD_VERSION_MAJOR*100 + KMD_VERSION_MINOR */

/* Diagnostic: which kernel the last fused launch on this host thread used
 * (0 none, 1 v1 direct (k > 13), 2 v2 warp-specialised (W % 4 != 0 or
 * unaligned), 3 v3 TMA with runtime M, 100 + M v3 TMA compiled for that M,
 * 150 + M the same with the albedo epilogue).  Lets the tests prove which
 * kernel they exercised.                                                    */
int32_t kmd_last_kernel(void);

#ifdef __cplusplus
}
#endif
#endif /* KMD_H */
