/*
 * kmd_oracle.h -- plain, slow, obviously-correct CPU oracle for the
 * kernel-map decoder + per-pixel filtering + kernel fusion of
 * arXiv 2202.05977 ("weight sharing kernel prediction").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_2202_05977_b200/, include/kmd.h) never links,
 * includes or calls anything here, and nothing here includes the product
 * headers: the two implementations share no code.
 *
 * Arithmetic: fp64 throughout (inputs are fp32, as the GPU path takes them).
 * Every function follows PAPER.md's equations literally, in the paper's
 * order (the "explicit kernel map" form of KPCN):
 *   unfold (Fig. 3)  ->  softmax along the channel axis (Eq. 3)
 *   -> apply the same weights to R, G, B (Eq. 4)
 *   -> per-pixel softmax fusion of the M filtered images (Eq. 5).
 * Readings of points the paper leaves open are DESIGN.md "Readings" R1-R16;
 * the ones used here: clamp-to-edge sampling for both the unfold and the
 * colour taps (R1), per-window max subtraction inside the softmax (R2, a
 * mathematically exact rewrite of Eq. 3), odd sizes only (R3), map i <->
 * sizes[i] (R4), blend given as logits and softmax-normalised inside (R5).
 *
 * Layout (all planar, row-major, contiguous, host memory):
 *   radiance   [N,3,H,W]  float     noisy demodulated HDR irradiance r(q)
 *   importance [N,M,H,W]  float     importance maps I_i(q)          (Eq. 2)
 *   blend      [N,M,H,W]  float     fusion logits (or alphas)       (Eq. 5)
 *   out        [N,3,rows,W] double  fused result  R^(p)
 */
#ifndef KMD_ORACLE_H
#define KMD_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    KMDO_OK = 0,
    KMDO_ERR_NULL = 1,    /* a required pointer is NULL                        */
    KMDO_ERR_CONFIG = 2,  /* even k, k < 1, M < 1, k > min(H,W)                 */
    KMDO_ERR_DIM = 3,     /* N,H,W < 1 or a row/pixel index out of range        */
    KMDO_ERR_NOMEM = 4
};

/* Fig. 3 / PAPER.md:232-234: unfold a single-channel H x W map with a k x k
 * sliding window.  out[(y*W+x)*k*k + j] = imap[clamp(y+dy), clamp(x+dx)],
 * offsets (dy,dx) = (j/k - r, j%k - r), r = (k-1)/2, row-major from (-r,-r). */
int kmdo_unfold(const float* imap, int32_t H, int32_t W, int32_t k, double* out);

/* Eq. 3 + "normalize it with a softmax function along the
 * channel axis": kmap[(y*W+x)*k*k + j] = w_p(q_j). */
int kmdo_kernel_map(const float* imap, int32_t H, int32_t W, int32_t k, double* kmap);

/* Eq. 4: R(p,c) = sum_j w_p(q_j) r_c(q_j), the same
 * weights for each colour channel.  radiance [3,H,W], out [3,H,W]. */
int kmdo_apply(const double* kmap, int32_t k, const float* radiance,
               int32_t H, int32_t W, double* out);

/* Eq. 5 with alpha = per-pixel softmax of the M logits
 * (PAPER.md:251).  filtered [M,3,H,W], blend [M,H,W] (may be NULL iff M==1),
 * out [3,H,W].  blend_is_logits == 0: blend already holds alpha_i(p). */
int kmdo_fuse(const double* filtered, const float* blend, int32_t M,
              int32_t H, int32_t W, int32_t blend_is_logits, double* out);

/* The whole reconstruction (unfold -> Eq. 3 -> Eq. 4 -> Eq. 5) evaluated one
 * output pixel at a time, each pixel's k x k kernel built on the fly (the
 * H x W x k^2 map never exists, so full 4K frames fit in host memory).
 * Computes output rows [y_begin, y_end) of every frame:
 *   out[((n*3 + c)*(y_end-y_begin) + (y-y_begin))*W + x].
 * threads <= 0: OpenMP default (all cores of the affinity mask). */
int kmdo_decode_filter_fuse_rows(const float* radiance, const float* importance,
                                 const float* blend, int32_t N, int32_t H, int32_t W,
                                 int32_t M, const int32_t* sizes, int32_t blend_is_logits,
                                 int32_t y_begin, int32_t y_end, int32_t threads,
                                 double* out);

/* Same, for an explicit list of pixels (frame n[t], row y[t], column x[t]);
 * out[t*3 + c].  Used to check sampled outputs of full-size frames. */
/* The same with the radiance in fp64 (the multi-resolution oracle filters
 * its fp64 pyramid levels D^l(r) without rounding them). */
int kmdo_decode_filter_fuse_rows_f64rad(const double* radiance, const float* importance,
                                        const float* blend, int32_t N, int32_t H, int32_t W,
                                        int32_t M, const int32_t* sizes, int32_t blend_is_logits,
                                        int32_t y_begin, int32_t y_end, int32_t threads,
                                        double* out);
int kmdo_decode_filter_fuse_pixels(const float* radiance, const float* importance,
                                   const float* blend, int32_t N, int32_t H, int32_t W,
                                   int32_t M, const int32_t* sizes, int32_t blend_is_logits,
                                   const int32_t* n, const int32_t* y, const int32_t* x,
                                   int64_t count, int32_t threads, double* out);

/* Albedo demodulation ("filter the noisy input
 * irradiance without albedo"): out[t] = radiance[t] / max(albedo[t], eps). */
int kmdo_demodulate(const float* radiance, const float* albedo, double eps, int64_t count, double* out);

/* Remodulation (Fig. 1 "multiply back the
 * albedo"): out[t] = irradiance[t] * albedo[t]. */
int kmdo_remodulate(const double* irradiance, const float* albedo, int64_t count, double* out);

/* ---- multi-resolution "Ours MR" (§5.2, Eq. 7) ----------
 * D: 2x2 mean downsampling: in [P][H][W] -> out [P][H/2][W/2]. */
int kmdo_downsample_2x2(const float* in, int64_t planes, int32_t H, int32_t W, double* out);
/* U: nearest upsampling: in [P][h][w] (fp64) -> out [P][2h][2w]. */
int kmdo_upsample_nearest(const double* in, int64_t planes, int32_t h, int32_t w, double* out);
/* Eq. 7: out = fine - alpha * U(D(fine)) + alpha * U(coarse),
 * fine [N][3][H][W] (fp64), coarse [N][3][H/2][W/2] (fp64), alpha [N][H][W]. */
int kmdo_combine_resolutions(const double* fine, const double* coarse, const float* alpha, int32_t N,
                             int32_t H, int32_t W, double* out);

/* ---- backward (NEXT row 3; Eq. 1) ----
 * Chain rule of Eq. 3 -> 4 -> 5 in the explicit-kernel form, one output pixel
 * at a time (serial):  with G = grad_out(p), alpha = softmax(B(p)),
 *   grad_blend_i(p)   = alpha_i sum_c G_c (R_i,c - Rhat_c)   (logits)
 *                     = sum_c G_c R_i,c                      (alpha given; 0 when M == 1)
 *   grad_imp_i(q_j)  += w_j sum_c alpha_i G_c (r_c(q_j) - R_i,c)   for every tap j of p's window
 * (dR/du_j of a softmax-weighted mean is w_j (r(q_j) - R); u_j = I_i(q_j)).
 * grad_out [N,3,H,W] fp64; grad_imp [N,M,H,W]; grad_blend [N,M,H,W] or NULL. */
int kmdo_backward(const float* radiance, const float* importance, const float* blend,
                  const double* grad_out, int32_t N, int32_t H, int32_t W, int32_t M,
                  const int32_t* sizes, int32_t blend_is_logits, double* grad_imp,
                  double* grad_blend);

/* ---- NEXT row 4: temporal accumulation pre-pass (§4.1;
 * SPEC.md:147-175).  Per pixel p = (x, y) of frame n, in the SPEC's order:
 *   reproject   s = nearest pixel of (x + mx, y + my), motion = (mx, my) in pixels
 *               (channel 0 = x); the nearest pixel of v is floor(v + 0.5), taken
 *               in fp32 as fx = floorf(((float)x + mx) + 0.5f) (reading R21);
 *               in_bounds = s inside the frame and prev_valid(s) != 0.
 *   consistency (fp32 decision, reading R22; no FMA contraction):
 *               d = cur_pos(p) - prev_pos(s);  pass_pos = (d0*d0 + d1*d1) + d2*d2 < pos_tol*pos_tol
 *               a = 2 cur_nrm(p) - 1, b = 2 prev_nrm(s) - 1   ([0,1] -> [-1,1]);
 *               pass_n = (a0*b0 + a1*b1) + a2*b2 > normal_tol * sqrtf(((a.a) * (b.b)))
 *   accumulate  mask = in_bounds && pass_pos && pass_n;
 *               accum = mask ? (1 - alpha) prev_rad(s) + alpha cur_rad(p) : cur_rad(p)   (fp64)
 * Layout: rad / pos / nrm [N,3,H,W] float, motion [N,2,H,W] float,
 * prev_valid and mask [N,H,W] uint8, accum [N,3,H,W] double. */
int kmdo_temporal_accumulate(const float* cur_rad, const float* prev_rad, const float* prev_pos,
                             const float* prev_nrm, const uint8_t* prev_valid, const float* cur_pos,
                             const float* cur_nrm, const float* motion, int32_t N, int32_t H, int32_t W,
                             float pos_tol, float normal_tol, float alpha, double* accum, uint8_t* mask);

/* Threads OpenMP would use for threads <= 0 (reported as cpu_baseline.cores). */
int kmdo_max_threads(void);

#ifdef __cplusplus
}
#endif
#endif
