/*
 * kmd_oracle.c -- CPU oracle (fp64) for arXiv 2202.05977's reconstruction
 * phase: kernel construction (unfold + softmax), filtering, kernel fusion.
 *
 * TEST INFRASTRUCTURE ONLY (see kmd_oracle.h).  Plain loops, no blocking,
 * no fusion beyond what the equations state, no use of the ratio-of-box
 * identity the GPU path relies on.  Each step cites the passage it follows.
 *
 * Pinned by tests/test_oracle_pins.py (scipy box filters, closed forms,
 * 50-digit mpmath brute force, invariants, a hand-worked example).
 */
#include "kmd_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

static int check_size(int32_t k, int32_t H, int32_t W) {
    /* Odd sizes only (R3: PAPER.md:251 says "even-sized" but lists
     * {3,5,7,...}; k_b = 3, k_s = 2 at PAPER.md:324).  k <= min(H,W) per
     * SPEC.md:231 (R12). */
    if (k < 1 || (k % 2) == 0 || k > H || k > W) return KMDO_ERR_CONFIG;
    return KMDO_OK;
}

/* ---- Step 1: unfold (Fig. 3; §4.2) -------
 * "we first unfold the importance map with a sliding window with window size
 * k to obtain the unnormalized kernel map with resolution H x W x (k*k)".
 * Channel j of pixel p=(y,x) holds I(q_j), q_j = p + (j/k - r, j%k - r),
 * clamped to the image (R1). */
static void window_taps(int H, int W, int k, int y, int x, int* qy, int* qx) {
    const int r = (k - 1) / 2;
    for (int j = 0; j < k * k; ++j) {
        const int dy = j / k - r, dx = j % k - r;
        qy[j] = clampi(y + dy, 0, H - 1);
        qx[j] = clampi(x + dx, 0, W - 1);
    }
}

static void unfold_pixel(const float* imap, int H, int W, int k, int y, int x,
                         double* u /* k*k */, int* qy /* k*k */, int* qx /* k*k */) {
    window_taps(H, W, k, y, x, qy, qx);
    for (int j = 0; j < k * k; ++j) u[j] = (double)imap[(size_t)qy[j] * W + qx[j]];
}

/* ---- Step 2: softmax along the channel axis (Eq. 3) ---
 * w_p(q) = exp(I(q)) / sum_{q' in Omega_p} exp(I(q')).
 * Computed as exp(u_j - m) / sum exp(u_j' - m) with m = max_j u_j, which is
 * the same number in exact arithmetic (R2) and keeps exp finite. */
static void softmax_window(const double* u, int kk, double* w) {
    double m = u[0];
    for (int j = 1; j < kk; ++j)
        if (u[j] > m) m = u[j];
    double s = 0.0;
    for (int j = 0; j < kk; ++j) {
        w[j] = exp(u[j] - m);
        s += w[j];
    }
    for (int j = 0; j < kk; ++j) w[j] = w[j] / s;
}

/* ---- Step 3: apply (Eq. 4) ----------------------------
 * R(p) = sum_q w_p(q) r(q), "the same weights to each RGB color channel". */
/* the radiance of one frame as fp32 (the inputs) or fp64 (a downsampled
 * pyramid level of the multi-resolution variant, kept in fp64) */
typedef struct {
    const float* f;
    const double* d;
} rad_t;
static double rad_at(rad_t r, size_t i) { return r.d ? r.d[i] : (double)r.f[i]; }
static rad_t rad_f32(const float* f) {
    rad_t r = {f, NULL};
    return r;
}
static rad_t rad_offset(rad_t r, size_t off) {
    rad_t o = r;
    if (o.d) o.d += off; else o.f += off;
    return o;
}

static void apply_window(const double* w, const int* qy, const int* qx, int kk,
                         rad_t radiance /* [3,H,W] */, int H, int W, double R[3]) {
    const size_t plane = (size_t)H * W;
    for (int c = 0; c < 3; ++c) {
        double acc = 0.0;
        for (int j = 0; j < kk; ++j)
            acc += w[j] * rad_at(radiance, c * plane + (size_t)qy[j] * W + qx[j]);
        R[c] = acc;
    }
}

/* ---- Step 4: fuse (Eq. 5; alpha softmax PAPER.md:251) --
 * R^(p) = sum_i alpha_i(p) R^{k_i}(p), 0 <= alpha_i <= 1, sum_i alpha_i = 1,
 * alpha = softmax over the M network output channels at p (R5),
 * again with the max subtracted (R2).  M == 1: alpha_0 = 1 (R11). */
static void fuse_pixel(const double* Ri /* [M][3] */, const double* b /* [M] or NULL */,
                       int M, int blend_is_logits, double out[3]) {
    double alpha[64];
    if (M == 1) {
        alpha[0] = 1.0;
    } else if (blend_is_logits) {
        double beta = b[0];
        for (int i = 1; i < M; ++i)
            if (b[i] > beta) beta = b[i];
        double s = 0.0;
        for (int i = 0; i < M; ++i) {
            alpha[i] = exp(b[i] - beta);
            s += alpha[i];
        }
        for (int i = 0; i < M; ++i) alpha[i] = alpha[i] / s;
    } else {
        for (int i = 0; i < M; ++i) alpha[i] = b[i];
    }
    for (int c = 0; c < 3; ++c) {
        double acc = 0.0;
        for (int i = 0; i < M; ++i) acc += alpha[i] * Ri[i * 3 + c];
        out[c] = acc;
    }
}

/* ======================= explicit-map entry points ======================= */

int kmdo_unfold(const float* imap, int32_t H, int32_t W, int32_t k, double* out) {
    if (!imap || !out) return KMDO_ERR_NULL;
    if (H < 1 || W < 1) return KMDO_ERR_DIM;
    int st = check_size(k, H, W);
    if (st) return st;
    const int kk = k * k;
    int* qy = (int*)malloc(sizeof(int) * kk);
    int* qx = (int*)malloc(sizeof(int) * kk);
    if (!qy || !qx) { free(qy); free(qx); return KMDO_ERR_NOMEM; }
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x)
            unfold_pixel(imap, H, W, k, y, x, out + ((size_t)y * W + x) * kk, qy, qx);
    free(qy); free(qx);
    return KMDO_OK;
}

int kmdo_kernel_map(const float* imap, int32_t H, int32_t W, int32_t k, double* kmap) {
    int st = kmdo_unfold(imap, H, W, k, kmap);
    if (st) return st;
    const int kk = k * k;
    double* w = (double*)malloc(sizeof(double) * kk);
    if (!w) return KMDO_ERR_NOMEM;
    for (size_t p = 0; p < (size_t)H * W; ++p) {
        softmax_window(kmap + p * kk, kk, w);
        memcpy(kmap + p * kk, w, sizeof(double) * kk);
    }
    free(w);
    return KMDO_OK;
}

int kmdo_apply(const double* kmap, int32_t k, const float* radiance,
               int32_t H, int32_t W, double* out) {
    if (!kmap || !radiance || !out) return KMDO_ERR_NULL;
    if (H < 1 || W < 1) return KMDO_ERR_DIM;
    int st = check_size(k, H, W);
    if (st) return st;
    const int kk = k * k;
    const size_t plane = (size_t)H * W;
    int* qy = (int*)malloc(sizeof(int) * kk);
    int* qx = (int*)malloc(sizeof(int) * kk);
    if (!qy || !qx) { free(qy); free(qx); return KMDO_ERR_NOMEM; }
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            double R[3];
            window_taps(H, W, k, y, x, qy, qx);      /* the q_j of Step 1 */
            apply_window(kmap + ((size_t)y * W + x) * kk, qy, qx, kk, rad_f32(radiance), H, W, R);
            for (int c = 0; c < 3; ++c) out[c * plane + (size_t)y * W + x] = R[c];
        }
    free(qy); free(qx);
    return KMDO_OK;
}

int kmdo_fuse(const double* filtered, const float* blend, int32_t M,
              int32_t H, int32_t W, int32_t blend_is_logits, double* out) {
    if (!filtered || !out) return KMDO_ERR_NULL;
    if (M < 1 || M > 64) return KMDO_ERR_CONFIG;
    if (M > 1 && !blend) return KMDO_ERR_NULL;
    if (H < 1 || W < 1) return KMDO_ERR_DIM;
    const size_t plane = (size_t)H * W;
    for (size_t p = 0; p < plane; ++p) {
        double Ri[64 * 3], b[64], o[3];
        for (int i = 0; i < M; ++i) {
            for (int c = 0; c < 3; ++c) Ri[i * 3 + c] = filtered[((size_t)i * 3 + c) * plane + p];
            b[i] = blend ? (double)blend[(size_t)i * plane + p] : 0.0;
        }
        fuse_pixel(Ri, b, M, blend_is_logits, o);
        for (int c = 0; c < 3; ++c) out[c * plane + p] = o[c];
    }
    return KMDO_OK;
}

/* ===================== streaming (per-pixel) entry points ================ */

static int check_all(const void* radiance, const float* importance, const float* blend,
                     int32_t N, int32_t H, int32_t W, int32_t M, const int32_t* sizes) {
    if (!radiance || !importance || !sizes) return KMDO_ERR_NULL;
    if (M < 1 || M > 64) return KMDO_ERR_CONFIG;
    if (M > 1 && !blend) return KMDO_ERR_NULL;
    if (N < 1 || H < 1 || W < 1) return KMDO_ERR_DIM;
    for (int i = 0; i < M; ++i) {
        int st = check_size(sizes[i], H, W);
        if (st) return st;
    }
    return KMDO_OK;
}

typedef struct {
    double *u, *w, *Ri;
    int *qy, *qx;
} scratch_t;

static int scratch_alloc(scratch_t* s, int M, const int32_t* sizes) {
    int kkmax = 1;
    for (int i = 0; i < M; ++i)
        if (sizes[i] * sizes[i] > kkmax) kkmax = sizes[i] * sizes[i];
    s->u = (double*)malloc(sizeof(double) * kkmax);
    s->w = (double*)malloc(sizeof(double) * kkmax);
    s->Ri = (double*)malloc(sizeof(double) * 3 * M);
    s->qy = (int*)malloc(sizeof(int) * kkmax);
    s->qx = (int*)malloc(sizeof(int) * kkmax);
    return (s->u && s->w && s->Ri && s->qy && s->qx) ? KMDO_OK : KMDO_ERR_NOMEM;
}

static void scratch_free(scratch_t* s) {
    free(s->u); free(s->w); free(s->Ri); free(s->qy); free(s->qx);
}

/* One output pixel: Steps 1-4 in the paper's order, for each size k_i. */
static void pixel(rad_t radiance, const float* importance, const float* blend,
                  int H, int W, int M, const int32_t* sizes, int blend_is_logits,
                  int n, int y, int x, scratch_t* s, double out[3]) {
    const size_t plane = (size_t)H * W;
    for (int i = 0; i < M; ++i) {
        const int k = sizes[i], kk = k * k;          /* map i <-> sizes[i] (R4) */
        const float* Ii = importance + ((size_t)n * M + i) * plane;
        unfold_pixel(Ii, H, W, k, y, x, s->u, s->qy, s->qx);          /* Fig. 3  */
        softmax_window(s->u, kk, s->w);                                /* Eq. 3   */
        apply_window(s->w, s->qy, s->qx, kk, rad_offset(radiance, (size_t)n * 3 * plane),
                     H, W, s->Ri + 3 * i);                             /* Eq. 4   */
    }
    double b[64];
    for (int i = 0; i < M; ++i)
        b[i] = blend ? (double)blend[((size_t)n * M + i) * plane + (size_t)y * W + x] : 0.0;
    fuse_pixel(s->Ri, b, M, blend_is_logits, out);                     /* Eq. 5   */
}

static int rows_impl(rad_t radiance, const float* importance,
                     const float* blend, int32_t N, int32_t H, int32_t W,
                     int32_t M, const int32_t* sizes, int32_t blend_is_logits,
                     int32_t y_begin, int32_t y_end, int32_t threads,
                     double* out) {
    if (!out) return KMDO_ERR_NULL;
    int st = check_all(radiance.f ? (const void*)radiance.f : (const void*)radiance.d, importance, blend, N, H, W,
                       M, sizes);
    if (st) return st;
    if (y_begin < 0 || y_end > H || y_begin > y_end) return KMDO_ERR_DIM;
    const int rows = y_end - y_begin;
    const long total = (long)N * rows;
    int err = KMDO_OK;
#ifdef _OPENMP
    const int nt = threads > 0 ? threads : omp_get_max_threads();
#pragma omp parallel num_threads(nt)
#endif
    {
        scratch_t s;
        int lst = scratch_alloc(&s, M, sizes);
        if (lst) {
#ifdef _OPENMP
#pragma omp atomic write
#endif
            err = lst;
        } else {
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
            for (long t = 0; t < total; ++t) {
                const int n = (int)(t / rows), yy = (int)(t % rows), y = y_begin + yy;
                for (int x = 0; x < W; ++x) {
                    double o[3];
                    pixel(radiance, importance, blend, H, W, M, sizes, blend_is_logits,
                          n, y, x, &s, o);
                    for (int c = 0; c < 3; ++c)
                        out[(((size_t)n * 3 + c) * rows + yy) * W + x] = o[c];
                }
            }
        }
        scratch_free(&s);
    }
    return err;
}

int kmdo_decode_filter_fuse_rows(const float* radiance, const float* importance,
                                 const float* blend, int32_t N, int32_t H, int32_t W,
                                 int32_t M, const int32_t* sizes, int32_t blend_is_logits,
                                 int32_t y_begin, int32_t y_end, int32_t threads,
                                 double* out) {
    rad_t r = {radiance, NULL};
    return rows_impl(r, importance, blend, N, H, W, M, sizes, blend_is_logits, y_begin, y_end, threads, out);
}

int kmdo_decode_filter_fuse_rows_f64rad(const double* radiance, const float* importance,
                                        const float* blend, int32_t N, int32_t H, int32_t W,
                                        int32_t M, const int32_t* sizes, int32_t blend_is_logits,
                                        int32_t y_begin, int32_t y_end, int32_t threads,
                                        double* out) {
    rad_t r = {NULL, radiance};
    return rows_impl(r, importance, blend, N, H, W, M, sizes, blend_is_logits, y_begin, y_end, threads, out);
}

int kmdo_decode_filter_fuse_pixels(const float* radiance, const float* importance,
                                   const float* blend, int32_t N, int32_t H, int32_t W,
                                   int32_t M, const int32_t* sizes, int32_t blend_is_logits,
                                   const int32_t* n, const int32_t* y, const int32_t* x,
                                   int64_t count, int32_t threads, double* out) {
    if (!out || !n || !y || !x) return KMDO_ERR_NULL;
    const rad_t rf = {radiance, NULL};
    int st = check_all(radiance, importance, blend, N, H, W, M, sizes);
    if (st) return st;
    for (int64_t t = 0; t < count; ++t)
        if (n[t] < 0 || n[t] >= N || y[t] < 0 || y[t] >= H || x[t] < 0 || x[t] >= W)
            return KMDO_ERR_DIM;
    int err = KMDO_OK;
#ifdef _OPENMP
    const int nt = threads > 0 ? threads : omp_get_max_threads();
#pragma omp parallel num_threads(nt)
#endif
    {
        scratch_t s;
        int lst = scratch_alloc(&s, M, sizes);
        if (lst) {
#ifdef _OPENMP
#pragma omp atomic write
#endif
            err = lst;
        } else {
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 64)
#endif
            for (int64_t t = 0; t < count; ++t)
                pixel(rf, importance, blend, H, W, M, sizes, blend_is_logits,
                      n[t], y[t], x[t], &s, out + 3 * t);
        }
        scratch_free(&s);
    }
    return err;
}

/* ---- albedo demodulation / remodulation */
int kmdo_demodulate(const float* radiance, const float* albedo, double eps, int64_t count, double* out) {
    if (!radiance || !albedo || !out) return KMDO_ERR_NULL;
    if (!(eps > 0.0)) return KMDO_ERR_CONFIG;
    for (int64_t t = 0; t < count; ++t) {
        const double a = (double)albedo[t];
        out[t] = (double)radiance[t] / (a > eps ? a : eps);
    }
    return KMDO_OK;
}

int kmdo_remodulate(const double* irradiance, const float* albedo, int64_t count, double* out) {
    if (!irradiance || !albedo || !out) return KMDO_ERR_NULL;
    for (int64_t t = 0; t < count; ++t) out[t] = irradiance[t] * (double)albedo[t];
    return KMDO_OK;
}

/* ---- multi-resolution (Eq. 7) -- */
int kmdo_downsample_2x2(const float* in, int64_t planes, int32_t H, int32_t W, double* out) {
    if (!in || !out) return KMDO_ERR_NULL;
    if (H < 2 || W < 2 || (H % 2) || (W % 2)) return KMDO_ERR_DIM;
    const int h = H / 2, w = W / 2;
    for (int64_t p = 0; p < planes; ++p)
        for (int y = 0; y < h; ++y)
            for (int x = 0; x < w; ++x) {
                const float* s = in + ((size_t)p * H + 2 * y) * W + 2 * x;
                /* arithmetic mean of the 2x2 source block */
                out[((size_t)p * h + y) * w + x] =
                    ((double)s[0] + (double)s[1] + (double)s[W] + (double)s[W + 1]) / 4.0;
            }
    return KMDO_OK;
}

int kmdo_upsample_nearest(const double* in, int64_t planes, int32_t h, int32_t w, double* out) {
    if (!in || !out) return KMDO_ERR_NULL;
    if (h < 1 || w < 1) return KMDO_ERR_DIM;
    const int H = 2 * h, W = 2 * w;
    for (int64_t p = 0; p < planes; ++p)
        for (int y = 0; y < H; ++y)
            for (int x = 0; x < W; ++x)
                out[((size_t)p * H + y) * W + x] = in[((size_t)p * h + y / 2) * w + x / 2];
    return KMDO_OK;
}

int kmdo_combine_resolutions(const double* fine, const double* coarse, const float* alpha, int32_t N,
                             int32_t H, int32_t W, double* out) {
    if (!fine || !coarse || !alpha || !out) return KMDO_ERR_NULL;
    if (N < 1 || H < 2 || W < 2 || (H % 2) || (W % 2)) return KMDO_ERR_DIM;
    const size_t plane = (size_t)H * W, cplane = plane / 4;
    const int h = H / 2, w = W / 2;
    double* dfine = (double*)malloc(sizeof(double) * cplane);
    double* udf = (double*)malloc(sizeof(double) * plane);
    double* uc = (double*)malloc(sizeof(double) * plane);
    if (!dfine || !udf || !uc) { free(dfine); free(udf); free(uc); return KMDO_ERR_NOMEM; }
    for (int n = 0; n < N; ++n)
        for (int c = 0; c < 3; ++c) {
            const double* f = fine + ((size_t)n * 3 + c) * plane;
            /* D(fine): the 2x2 mean, in fp64 */
            for (int y = 0; y < h; ++y)
                for (int x = 0; x < w; ++x)
                    dfine[(size_t)y * w + x] = (f[(size_t)2 * y * W + 2 * x] + f[(size_t)2 * y * W + 2 * x + 1] +
                                                f[(size_t)(2 * y + 1) * W + 2 * x] +
                                                f[(size_t)(2 * y + 1) * W + 2 * x + 1]) / 4.0;
            kmdo_upsample_nearest(dfine, 1, h, w, udf);
            kmdo_upsample_nearest(coarse + ((size_t)n * 3 + c) * cplane, 1, h, w, uc);
            const float* a = alpha + (size_t)n * plane;
            double* o = out + ((size_t)n * 3 + c) * plane;
            for (size_t q = 0; q < plane; ++q) o[q] = f[q] - (double)a[q] * udf[q] + (double)a[q] * uc[q];
        }
    free(dfine); free(udf); free(uc);
    return KMDO_OK;
}

/* ---- backward (NEXT row 3) ---------------------------------------------- */
int kmdo_backward(const float* radiance, const float* importance, const float* blend,
                  const double* grad_out, int32_t N, int32_t H, int32_t W, int32_t M,
                  const int32_t* sizes, int32_t blend_is_logits, double* grad_imp,
                  double* grad_blend) {
    if (!grad_out || !grad_imp) return KMDO_ERR_NULL;
    int st = check_all(radiance, importance, blend, N, H, W, M, sizes);
    if (st) return st;
    const size_t plane = (size_t)H * W;
    memset(grad_imp, 0, sizeof(double) * (size_t)N * M * plane);
    if (grad_blend) memset(grad_blend, 0, sizeof(double) * (size_t)N * M * plane);
    scratch_t s;
    st = scratch_alloc(&s, M, sizes);
    if (st) { scratch_free(&s); return st; }
    int kkmax = 1;
    for (int i = 0; i < M; ++i)
        if (sizes[i] * sizes[i] > kkmax) kkmax = sizes[i] * sizes[i];
    double* wall = (double*)malloc(sizeof(double) * (size_t)M * kkmax);  /* w of every size */
    int* qyall = (int*)malloc(sizeof(int) * (size_t)M * kkmax);
    int* qxall = (int*)malloc(sizeof(int) * (size_t)M * kkmax);
    if (!wall || !qyall || !qxall) { free(wall); free(qyall); free(qxall); scratch_free(&s); return KMDO_ERR_NOMEM; }
    for (int n = 0; n < N; ++n)
        for (int y = 0; y < H; ++y)
            for (int x = 0; x < W; ++x) {
                const float* rad = radiance + (size_t)n * 3 * plane;
                /* forward, Steps 1-3 per size (as pixel()) keeping the weights */
                for (int i = 0; i < M; ++i) {
                    const int k = sizes[i], kk = k * k;
                    const float* Ii = importance + ((size_t)n * M + i) * plane;
                    unfold_pixel(Ii, H, W, k, y, x, s.u, qyall + i * kkmax, qxall + i * kkmax);
                    softmax_window(s.u, kk, wall + i * kkmax);
                    apply_window(wall + i * kkmax, qyall + i * kkmax, qxall + i * kkmax, kk, rad_f32(rad), H, W,
                                 s.Ri + 3 * i);
                }
                /* Step 4 weights */
                double alpha[64], b[64];
                for (int i = 0; i < M; ++i)
                    b[i] = blend ? (double)blend[((size_t)n * M + i) * plane + (size_t)y * W + x] : 0.0;
                if (M == 1) {
                    alpha[0] = 1.0;
                } else if (blend_is_logits) {
                    double beta = b[0], sum = 0.0;
                    for (int i = 1; i < M; ++i) if (b[i] > beta) beta = b[i];
                    for (int i = 0; i < M; ++i) { alpha[i] = exp(b[i] - beta); sum += alpha[i]; }
                    for (int i = 0; i < M; ++i) alpha[i] /= sum;
                } else {
                    for (int i = 0; i < M; ++i) alpha[i] = b[i];
                }
                double Rh[3] = {0, 0, 0};
                for (int i = 0; i < M; ++i)
                    for (int c = 0; c < 3; ++c) Rh[c] += alpha[i] * s.Ri[3 * i + c];
                double G[3];
                for (int c = 0; c < 3; ++c) G[c] = grad_out[((size_t)n * 3 + c) * plane + (size_t)y * W + x];
                for (int i = 0; i < M; ++i) {
                    const int kk = sizes[i] * sizes[i];
                    if (grad_blend && M > 1) {
                        double v = 0.0;
                        for (int c = 0; c < 3; ++c)
                            v += blend_is_logits ? alpha[i] * G[c] * (s.Ri[3 * i + c] - Rh[c]) : G[c] * s.Ri[3 * i + c];
                        grad_blend[((size_t)n * M + i) * plane + (size_t)y * W + x] = v;
                    }
                    double* gI = grad_imp + ((size_t)n * M + i) * plane;
                    for (int j = 0; j < kk; ++j) {
                        const int qy = qyall[i * kkmax + j], qx = qxall[i * kkmax + j];
                        double acc = 0.0;
                        for (int c = 0; c < 3; ++c)
                            acc += alpha[i] * G[c] * ((double)rad[c * plane + (size_t)qy * W + qx] - s.Ri[3 * i + c]);
                        gI[(size_t)qy * W + qx] += wall[i * kkmax + j] * acc;
                    }
                }
            }
    free(wall); free(qyall); free(qxall);
    scratch_free(&s);
    return KMDO_OK;
}

/* ---- temporal accumulation (NEXT row 4) ---------------------------------- */
int kmdo_temporal_accumulate(const float* cur_rad, const float* prev_rad, const float* prev_pos,
                             const float* prev_nrm, const uint8_t* prev_valid, const float* cur_pos,
                             const float* cur_nrm, const float* motion, int32_t N, int32_t H, int32_t W,
                             float pos_tol, float normal_tol, float alpha, double* accum, uint8_t* mask) {
    if (N < 0 || H < 0 || W < 0) return KMDO_ERR_DIM;
    if ((size_t)N * H * W == 0) return KMDO_OK;
    if (!cur_rad || !prev_rad || !prev_pos || !prev_nrm || !prev_valid || !cur_pos || !cur_nrm || !motion ||
        !accum || !mask)
        return KMDO_ERR_NULL;
    if (!(pos_tol > 0.0f) || !(normal_tol > 0.0f && normal_tol <= 1.0f) || !(alpha > 0.0f && alpha <= 1.0f))
        return KMDO_ERR_CONFIG;
    const size_t plane = (size_t)H * W;
    for (int n = 0; n < N; ++n)
        for (int y = 0; y < H; ++y)
            for (int x = 0; x < W; ++x) {
                const size_t p = (size_t)y * W + x;
                const float* cr = cur_rad + (size_t)n * 3 * plane;
                /* reproject (nearest pixel, fp32) */
                const float mx = motion[((size_t)n * 2 + 0) * plane + p];
                const float my = motion[((size_t)n * 2 + 1) * plane + p];
                const float fx = floorf(((float)x + mx) + 0.5f);
                const float fy = floorf(((float)y + my) + 0.5f);
                int in_bounds = fx >= 0.0f && fx <= (float)(W - 1) && fy >= 0.0f && fy <= (float)(H - 1);
                size_t s = 0;
                if (in_bounds) {
                    s = (size_t)(int)fy * W + (size_t)(int)fx;
                    in_bounds = prev_valid[(size_t)n * plane + s] != 0;
                }
                int m = 0;
                if (in_bounds) {
                    /* consistency test (fp32) */
                    const float* cp = cur_pos + (size_t)n * 3 * plane;
                    const float* pp = prev_pos + (size_t)n * 3 * plane;
                    const float* cn = cur_nrm + (size_t)n * 3 * plane;
                    const float* pn = prev_nrm + (size_t)n * 3 * plane;
                    float d[3], a[3], b[3];
                    for (int c = 0; c < 3; ++c) {
                        d[c] = cp[c * plane + p] - pp[c * plane + s];
                        a[c] = 2.0f * cn[c * plane + p] - 1.0f;
                        b[c] = 2.0f * pn[c * plane + s] - 1.0f;
                    }
                    const float d2 = (d[0] * d[0] + d[1] * d[1]) + d[2] * d[2];
                    const float pass_pos = d2 < pos_tol * pos_tol;
                    const float dot = (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2];
                    const float aa = (a[0] * a[0] + a[1] * a[1]) + a[2] * a[2];
                    const float bb = (b[0] * b[0] + b[1] * b[1]) + b[2] * b[2];
                    const int pass_n = dot > normal_tol * sqrtf(aa * bb);
                    m = pass_pos && pass_n;
                }
                mask[(size_t)n * plane + p] = (uint8_t)m;
                /* accumulate */
                for (int c = 0; c < 3; ++c) {
                    const double cur = cr[c * plane + p];
                    double v = cur;
                    if (m) v = (1.0 - (double)alpha) * (double)prev_rad[((size_t)n * 3 + c) * plane + s] + (double)alpha * cur;
                    accum[((size_t)n * 3 + c) * plane + p] = v;
                }
            }
    return KMDO_OK;
}

int kmdo_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
