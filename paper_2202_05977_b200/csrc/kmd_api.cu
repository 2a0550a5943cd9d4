// kmd_api.cu -- the extern "C" boundary of libkmd (declared in include/kmd.h).
// Argument checks are synchronous and precede every CUDA call; work is
// enqueued on the caller's stream.  No per-call allocation.
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "kmd_kernels.h"

namespace {
thread_local int g_last_kernel = 0;
thread_local int g_max_ctas = 0;  // grid cap for the next fused launches (multi-resolution concurrency)
}  // namespace
namespace kmd {
void set_last_kernel(int k) { g_last_kernel = k; }
}  // namespace kmd

namespace {

thread_local char g_err[512] = "";

kmd_status fail(kmd_status s, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return s;
}

}  // namespace

namespace kmd {
// the error detail of the other translation units (kmd_band.cu)
kmd_status api_fail(kmd_status s, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return s;
}
void api_clear_error() { g_err[0] = 0; }
}  // namespace kmd

namespace {

kmd_status cuda_fail(cudaError_t e, const char* what) {
    return fail(KMD_ERR_CUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

kmd_status check_cfg(const kmd_config* cfg, int64_t H, int64_t W) {
    if (!cfg) return fail(KMD_ERR_NULL, "cfg is NULL");
    if (cfg->num_sizes < 1 || cfg->num_sizes > KMD_MAX_SIZES)
        return fail(KMD_ERR_CONFIG, "num_sizes=%d not in [1,%d]", cfg->num_sizes, KMD_MAX_SIZES);
    for (int i = 0; i < cfg->num_sizes; ++i) {
        const int k = cfg->sizes[i];
        if (k < 1 || k % 2 == 0 || k > KMD_MAX_K)
            return fail(KMD_ERR_CONFIG, "sizes[%d]=%d must be odd and in [1,%d]", i, k, KMD_MAX_K);
        if (k > H || k > W)
            return fail(KMD_ERR_CONFIG, "sizes[%d]=%d exceeds min(H,W)=%lld", i, k,
                        (long long)(H < W ? H : W));
    }
    if (cfg->blend_is_logits != 0 && cfg->blend_is_logits != 1)
        return fail(KMD_ERR_CONFIG, "blend_is_logits=%d must be 0 or 1", cfg->blend_is_logits);
    if (cfg->border != KMD_BORDER_CLAMP)
        return fail(KMD_ERR_CONFIG, "border=%d unsupported (only KMD_BORDER_CLAMP)", cfg->border);
    return KMD_OK;
}

int rmax_of(const kmd_config* cfg) {
    int r = 0;
    for (int i = 0; i < cfg->num_sizes; ++i) r = r > (cfg->sizes[i] - 1) / 2 ? r : (cfg->sizes[i] - 1) / 2;
    return r;
}

bool overlaps(const void* a, size_t abytes, const void* b, size_t bbytes) {
    if (!a || !b || abytes == 0 || bbytes == 0) return false;
    const uintptr_t a0 = (uintptr_t)a, b0 = (uintptr_t)b;
    return a0 < b0 + bbytes && b0 < a0 + abytes;
}

// Common launch path for whole frames and bands.
// development switches / checked-build jitter seed (env KMD_DEBUG, read once)
int debug_env() {
    static const int dbg = [] { const char* e = getenv("KMD_DEBUG"); return e ? atoi(e) : 0; }();
    return dbg;
}

kmd_status run_fused(kmd::FusedParams p, const kmd_config* cfg, cudaStream_t stream) {
    p.M = cfg->num_sizes;
    p.rmax = rmax_of(cfg);
    p.blend_is_logits = cfg->blend_is_logits;
    for (int i = 0; i < KMD_MAX_SIZES; ++i) p.sizes[i] = i < cfg->num_sizes ? cfg->sizes[i] : 1;
    if (p.M == 1) p.blend = nullptr;  // softmax of one logit is 1 (reading R11)
    p.debug = debug_env();
    const size_t bplane = (size_t)p.buf_rows * p.W, oplane = (size_t)p.out_rows * p.W;
    const size_t esz = p.in16 ? 2 : 4;  // bytes per importance / logit element
    const int total = p.N;
    for (int n0 = 0; n0 < total; n0 += 65535) {
        kmd::FusedParams q = p;
        q.N = total - n0 < 65535 ? total - n0 : 65535;
        q.rad = p.rad + (size_t)n0 * 3 * bplane;
        q.imp = (const float*)((const char*)p.imp + (size_t)n0 * p.M * bplane * esz);
        q.blend = p.blend ? (const float*)((const char*)p.blend + (size_t)n0 * p.M * oplane * esz) : nullptr;
        q.out = p.out + (size_t)n0 * 3 * oplane;
        cudaError_t e;
        if (p.in16) {
            // bf16 inputs: the TMA kernel only (checked by the caller)
            if (!kmd::tma_supported(q)) return fail(KMD_ERR_ALIGN, "bf16 path needs W %% 8 == 0 and 16-byte aligned buffers");
            e = kmd::launch_fused_tma(q, stream);
        } else if (kmd::tma_supported(q)) {
            e = kmd::launch_fused_tma(q, stream);  // records its specialisation
        } else if (kmd::ws_supported(q)) {
            kmd::set_last_kernel(kmd::LK_WS);
            e = kmd::launch_fused_ws(q, stream);
        } else {
            kmd::set_last_kernel(kmd::LK_DIRECT);
            e = kmd::launch_fused_direct(q, stream);
        }
        if (e != cudaSuccess) return cuda_fail(e, "fused kernel launch");
    }
    return KMD_OK;
}

}  // namespace

extern "C" {

kmd_status kmd_decode_filter_fuse_remod(const float* radiance, const float* importance,
                                        const float* blend, const float* albedo, float* out,
                                        int32_t N, int32_t H, int32_t W, const kmd_config* cfg,
                                        kmd_stream_t stream) {
    g_err[0] = 0;
    if (N < 0) return fail(KMD_ERR_DIM, "N=%d < 0", N);
    if (N > 0 && (H < 1 || W < 1)) return fail(KMD_ERR_DIM, "H=%d, W=%d must be >= 1", H, W);
    if (!cfg) return fail(KMD_ERR_NULL, "cfg is NULL");
    if (N > 0) {
        kmd_status s = check_cfg(cfg, H, W);
        if (s) return s;
    }
    if (N == 0) return KMD_OK;  // no-op; pointers of empty tensors may be NULL
    if (!radiance || !importance || !out) return fail(KMD_ERR_NULL, "radiance/importance/out is NULL");
    if (cfg->num_sizes > 1 && !blend) return fail(KMD_ERR_NULL, "blend is NULL with M=%d > 1", cfg->num_sizes);
    const size_t plane = (size_t)H * W * sizeof(float);
    const size_t M = (size_t)cfg->num_sizes;
    if (overlaps(out, 3 * N * plane, radiance, 3 * N * plane) ||
        overlaps(out, 3 * N * plane, importance, M * N * plane) ||
        (M > 1 && overlaps(out, 3 * N * plane, blend, M * N * plane)) ||
        overlaps(out, 3 * N * plane, albedo, 3 * N * plane))
        return fail(KMD_ERR_ALIAS, "out overlaps an input");
    kmd::FusedParams p{};
    p.rad = radiance; p.imp = importance; p.blend = blend; p.out = out; p.albedo = albedo;
    p.max_ctas = g_max_ctas;
    p.N = N; p.W = W; p.H = H;
    p.row_base = 0; p.buf_rows = H; p.out_y0 = 0; p.out_rows = H;
    return run_fused(p, cfg, (cudaStream_t)stream);
}

kmd_status kmd_decode_filter_fuse(const float* radiance, const float* importance,
                                  const float* blend, float* out, int32_t N, int32_t H,
                                  int32_t W, const kmd_config* cfg, kmd_stream_t stream) {
    return kmd_decode_filter_fuse_remod(radiance, importance, blend, nullptr, out, N, H, W, cfg, stream);
}

kmd_status kmd_decode_filter_fuse_bf16(const float* radiance, const uint16_t* importance,
                                       const uint16_t* blend, float* out, int32_t N, int32_t H,
                                       int32_t W, const kmd_config* cfg, kmd_stream_t stream) {
    g_err[0] = 0;
    if (N < 0) return fail(KMD_ERR_DIM, "N=%d < 0", N);
    if (N > 0 && (H < 1 || W < 1)) return fail(KMD_ERR_DIM, "H=%d, W=%d must be >= 1", H, W);
    if (!cfg) return fail(KMD_ERR_NULL, "cfg is NULL");
    if (N > 0) {
        kmd_status s = check_cfg(cfg, H, W);
        if (s) return s;
    }
    if (N == 0) return KMD_OK;
    if (!radiance || !importance || !out) return fail(KMD_ERR_NULL, "radiance/importance/out is NULL");
    if (cfg->num_sizes > 1 && !blend) return fail(KMD_ERR_NULL, "blend is NULL with M=%d > 1", cfg->num_sizes);
    if (W % 8 != 0) return fail(KMD_ERR_ALIGN, "bf16 path needs W %% 8 == 0 (W=%d)", W);
    const uintptr_t a = (uintptr_t)radiance | (uintptr_t)importance | (uintptr_t)out |
                        (uintptr_t)(cfg->num_sizes > 1 ? blend : nullptr);
    if (a & 15) return fail(KMD_ERR_ALIGN, "bf16 path needs 16-byte aligned buffers");
    const size_t px = (size_t)H * W;
    const size_t M = (size_t)cfg->num_sizes;
    if (overlaps(out, 3 * N * px * 4, radiance, 3 * N * px * 4) ||
        overlaps(out, 3 * N * px * 4, importance, M * N * px * 2) ||
        (M > 1 && overlaps(out, 3 * N * px * 4, blend, M * N * px * 2)))
        return fail(KMD_ERR_ALIAS, "out overlaps an input");
    for (int k = 0; k < cfg->num_sizes; ++k)
        if ((cfg->sizes[k] - 1) / 2 > 6)
            return fail(KMD_ERR_CONFIG, "bf16 path supports sizes <= 13 (sizes[%d]=%d)", k, cfg->sizes[k]);
    kmd::FusedParams p{};
    p.rad = radiance;
    p.imp = reinterpret_cast<const float*>(importance);
    p.blend = reinterpret_cast<const float*>(blend);
    p.out = out;
    p.in16 = 1;
    p.max_ctas = g_max_ctas;
    p.N = N; p.W = W; p.H = H;
    p.row_base = 0; p.buf_rows = H; p.out_y0 = 0; p.out_rows = H;
    return run_fused(p, cfg, (cudaStream_t)stream);
}

kmd_status kmd_demodulate(const float* radiance, const float* albedo, float eps, float* irradiance,
                          int32_t N, int32_t H, int32_t W, kmd_stream_t stream) {
    g_err[0] = 0;
    if (N < 0 || (N > 0 && (H < 1 || W < 1))) return fail(KMD_ERR_DIM, "bad N/H/W");
    if (!(eps > 0.f)) return fail(KMD_ERR_CONFIG, "eps must be > 0");
    if (N == 0) return KMD_OK;
    if (!radiance || !albedo || !irradiance) return fail(KMD_ERR_NULL, "NULL buffer");
    const size_t bytes = (size_t)N * 3 * H * W * sizeof(float);
    if (overlaps(irradiance, bytes, albedo, bytes)) return fail(KMD_ERR_ALIAS, "irradiance overlaps albedo");
    cudaError_t e = kmd::launch_albedo_op(radiance, albedo, eps, irradiance, (long long)N * 3 * H * W, 0,
                                          (cudaStream_t)stream);
    return e == cudaSuccess ? KMD_OK : cuda_fail(e, "demodulate launch");
}

kmd_status kmd_remodulate(const float* irradiance, const float* albedo, float* out, int32_t N, int32_t H,
                          int32_t W, kmd_stream_t stream) {
    g_err[0] = 0;
    if (N < 0 || (N > 0 && (H < 1 || W < 1))) return fail(KMD_ERR_DIM, "bad N/H/W");
    if (N == 0) return KMD_OK;
    if (!irradiance || !albedo || !out) return fail(KMD_ERR_NULL, "NULL buffer");
    const size_t bytes = (size_t)N * 3 * H * W * sizeof(float);
    if (overlaps(out, bytes, albedo, bytes)) return fail(KMD_ERR_ALIAS, "out overlaps albedo");
    cudaError_t e = kmd::launch_albedo_op(irradiance, albedo, 0.f, out, (long long)N * 3 * H * W, 1,
                                          (cudaStream_t)stream);
    return e == cudaSuccess ? KMD_OK : cuda_fail(e, "remodulate launch");
}

kmd_status kmd_decode_filter(const float* radiance, const float* importance_i, float* out_i,
                             int32_t N, int32_t H, int32_t W, int32_t k, kmd_stream_t stream) {
    kmd_config cfg{};
    cfg.num_sizes = 1;
    cfg.sizes[0] = k;
    cfg.blend_is_logits = 1;
    cfg.border = KMD_BORDER_CLAMP;
    return kmd_decode_filter_fuse(radiance, importance_i, nullptr, out_i, N, H, W, &cfg, stream);
}

kmd_status kmd_fuse(const float* filtered, const float* blend, float* out, int32_t N, int32_t H,
                    int32_t W, int32_t M, int32_t blend_is_logits, kmd_stream_t stream) {
    g_err[0] = 0;
    if (N < 0) return fail(KMD_ERR_DIM, "N=%d < 0", N);
    if (N > 0 && (H < 1 || W < 1)) return fail(KMD_ERR_DIM, "H=%d, W=%d must be >= 1", H, W);
    if (M < 1 || M > KMD_MAX_SIZES) return fail(KMD_ERR_CONFIG, "M=%d not in [1,%d]", M, KMD_MAX_SIZES);
    if (blend_is_logits != 0 && blend_is_logits != 1)
        return fail(KMD_ERR_CONFIG, "blend_is_logits=%d must be 0 or 1", blend_is_logits);
    if (N == 0) return KMD_OK;
    if (!filtered || !out) return fail(KMD_ERR_NULL, "filtered/out is NULL");
    if (M > 1 && !blend) return fail(KMD_ERR_NULL, "blend is NULL with M=%d > 1", M);
    const size_t plane = (size_t)H * W * sizeof(float);
    if (overlaps(out, 3 * N * plane, filtered, 3 * (size_t)M * N * plane) ||
        (M > 1 && overlaps(out, 3 * N * plane, blend, (size_t)M * N * plane)))
        return fail(KMD_ERR_ALIAS, "out overlaps an input");
    cudaError_t e = kmd::launch_fuse_only(filtered, M > 1 ? blend : nullptr, out, N, H, W, M,
                                          blend_is_logits, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "fuse kernel launch");
    return KMD_OK;
}

}  // extern "C"

namespace {

// Validates a row band and fills its launch parameters (the checks of
// kmd_decode_filter_fuse_band).  Returns KMD_OK with *skip = true when N == 0.
kmd_status band_params(const float* radiance, const float* importance, const float* blend, float* out, int32_t N,
                       int32_t band_rows, int32_t W, int32_t halo_top, int32_t halo_bot, int32_t y0,
                       int32_t H_global, const kmd_config* cfg, kmd::FusedParams* p, bool* skip, int in16 = 0) {
    *skip = false;
    if (N < 0) return fail(KMD_ERR_DIM, "N=%d < 0", N);
    if (!cfg) return fail(KMD_ERR_NULL, "cfg is NULL");
    if (N > 0) {
        if (band_rows < 1 || W < 1 || H_global < 1)
            return fail(KMD_ERR_DIM, "band_rows=%d, W=%d, H_global=%d must be >= 1", band_rows, W, H_global);
        if (halo_top < 0 || halo_bot < 0 || y0 < 0 || y0 - halo_top < 0 ||
            (int64_t)y0 + band_rows + halo_bot > H_global)
            return fail(KMD_ERR_DIM, "band [%d-%d, %d+%d+%d) outside frame of %d rows", y0, halo_top,
                        y0, band_rows, halo_bot, H_global);
        kmd_status s = check_cfg(cfg, H_global, W);
        if (s) return s;
        const int r = rmax_of(cfg);
        const int need_top = r < y0 ? r : y0;
        const int below = H_global - y0 - band_rows;
        const int need_bot = r < below ? r : below;
        if (halo_top < need_top || halo_bot < need_bot)
            return fail(KMD_ERR_DIM, "halo (%d,%d) smaller than required (%d,%d) for r_max=%d", halo_top,
                        halo_bot, need_top, need_bot, r);
    }
    if (N == 0) {
        *skip = true;
        return KMD_OK;
    }
    if (!radiance || !importance || !out) return fail(KMD_ERR_NULL, "radiance/importance/out is NULL");
    if (cfg->num_sizes > 1 && !blend) return fail(KMD_ERR_NULL, "blend is NULL with M=%d > 1", cfg->num_sizes);
    const int buf_rows = halo_top + band_rows + halo_bot;
    const size_t bplane = (size_t)buf_rows * W * sizeof(float), oplane = (size_t)band_rows * W * sizeof(float);
    const size_t M = (size_t)cfg->num_sizes, esz = in16 ? 2 : 4;
    if (overlaps(out, 3 * N * oplane, radiance, 3 * N * bplane) ||
        overlaps(out, 3 * N * oplane, importance, M * N * bplane / 4 * esz) ||
        (M > 1 && overlaps(out, 3 * N * oplane, blend, M * N * oplane / 4 * esz)))
        return fail(KMD_ERR_ALIAS, "out overlaps an input");
    kmd::FusedParams q{};
    q.in16 = in16;
    q.rad = radiance; q.imp = importance; q.blend = blend; q.out = out;
    q.N = N; q.W = W; q.H = H_global;
    q.row_base = y0 - halo_top; q.buf_rows = buf_rows; q.out_y0 = y0; q.out_rows = band_rows;
    *p = q;
    return KMD_OK;
}

}  // namespace

extern "C" {

kmd_status kmd_decode_filter_fuse_band(const float* radiance, const float* importance,
                                       const float* blend, float* out, int32_t N,
                                       int32_t band_rows, int32_t W, int32_t halo_top,
                                       int32_t halo_bot, int32_t y0, int32_t H_global,
                                       const kmd_config* cfg, kmd_stream_t stream) {
    return kmd_decode_filter_fuse_band_part(radiance, importance, blend, out, N, band_rows, W, halo_top, halo_bot,
                                            y0, H_global, cfg, KMD_BAND_ALL, stream);
}

kmd_status kmd_decode_filter_fuse_band_part(const float* radiance, const float* importance,
                                            const float* blend, float* out, int32_t N,
                                            int32_t band_rows, int32_t W, int32_t halo_top,
                                            int32_t halo_bot, int32_t y0, int32_t H_global,
                                            const kmd_config* cfg, int32_t part, kmd_stream_t stream) {
    g_err[0] = 0;
    if (part != KMD_BAND_ALL && part != KMD_BAND_INTERIOR && part != KMD_BAND_SEAMS)
        return fail(KMD_ERR_CONFIG, "part=%d not one of KMD_BAND_ALL/INTERIOR/SEAMS", part);
    kmd::FusedParams p{};
    bool skip = false;
    kmd_status s = band_params(radiance, importance, blend, out, N, band_rows, W, halo_top, halo_bot, y0, H_global,
                               cfg, &p, &skip);
    if (s || skip) return s;
    if (part == KMD_BAND_ALL) return run_fused(p, cfg, (cudaStream_t)stream);
    // Interior / seam split on the TMA kernel's global tile grid: a tile row
    // is interior when every row its windows read is an owned row (or is
    // clamped at a frame edge that has no neighbour), so it can run before the
    // halo rows arrive; the seam tile rows are the rest.  Each tile is
    // computed once, by one of the two launches, in the same order as in the
    // whole-frame call (bitwise equal results).
    {
        kmd::FusedParams t = p;
        t.M = cfg->num_sizes;
        for (int i = 0; i < KMD_MAX_SIZES; ++i) t.sizes[i] = i < cfg->num_sizes ? cfg->sizes[i] : 1;
        if (!kmd::tma_supported(t))  // other kernels: no split, the seam part does the whole band
            return part == KMD_BAND_SEAMS ? run_fused(p, cfg, (cudaStream_t)stream) : KMD_OK;
    }
    const int TH = kmd::tma_tile_rows(), r = rmax_of(cfg);
    const int tile_begin = (y0 / TH) * TH;
    const int tiles_y = (y0 + band_rows - tile_begin + TH - 1) / TH;
    int k_lo = 0, k_hi = tiles_y;
    if (halo_top > 0)
        while (k_lo < tiles_y && tile_begin + k_lo * TH - r < y0) ++k_lo;
    if (halo_bot > 0)
        while (k_hi > 0 && tile_begin + (k_hi - 1) * TH + TH + r > y0 + band_rows) --k_hi;
    if (k_hi < k_lo) k_hi = k_lo;  // no interior tile row
    if (part == KMD_BAND_INTERIOR) {
        if (k_hi == k_lo) return KMD_OK;
        p.tile_y_begin = tile_begin + k_lo * TH;
        p.tile_rows_a = k_hi - k_lo;
        p.tile_rows_total = k_hi - k_lo;
    } else {
        const int total = k_lo + (tiles_y - k_hi);
        if (total == 0) return KMD_OK;
        p.tile_y_begin = tile_begin;
        p.tile_rows_a = k_lo;
        p.tile_y_begin_b = tile_begin + k_hi * TH;
        p.tile_rows_total = total;
    }
    return run_fused(p, cfg, (cudaStream_t)stream);
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Host entry point: each frame is cut into row bands; band b's rows (+ r_max
// halo rows) are copied host->device with one 3-D copy per tensor, processed by
// the band kernel and copied back, on three streams so the copy engines (H2D,
// D2H) and the SMs overlap across bands and frames.  The caller's stream is
// joined at the start and the end, so the call behaves as stream-ordered work.
namespace {

#ifndef KMD_HOST_BANDS
#define KMD_HOST_BANDS 2
#endif
#ifndef KMD_HOST_LASTW
#define KMD_HOST_LASTW 3  // weight of the last band (the others: 5)
#endif
constexpr int HOST_MAX_BANDS = KMD_HOST_BANDS;

struct HostBand {
    int y0, rows, top, bot;  // owned rows [y0, y0+rows), halo rows above/below
};

int host_bands(int H, int rmax, HostBand* out) {
    int nb = HOST_MAX_BANDS;
    while (nb > 1 && (int64_t)KMD_HOST_LASTW * H / (5 * (nb - 1) + KMD_HOST_LASTW) < 2 * rmax + 8) --nb;
    // Two bands, the last 3/5 of the first (KMD_HOST_BANDS, KMD_HOST_LASTW):
    // the call ends with the last band's kernel and D2H, which nothing
    // overlaps, while more, smaller copies lose PCIe throughput.  Measured
    // (1080p M = 6, consecutive calls): 4 bands 832 / 1292 Mpix/s (fp32 /
    // bf16 inputs), 3 bands 848 / 1328, 2 bands 5:2 871 / 1354, 2 bands 5:3
    // 874 / 1414, 2 bands 5:5 850 / 1369, 1 band 742 / 1094.
    const int64_t wsum = 5 * (nb - 1) + KMD_HOST_LASTW;
    auto edge = [&](int b) { return (int)(b == nb ? H : (int64_t)5 * b * H / wsum); };
    for (int b = 0; b < nb; ++b) {
        const int y0 = edge(b), y1 = edge(b + 1);
        out[b].y0 = y0;
        out[b].rows = y1 - y0;
        out[b].top = y0 < rmax ? y0 : rmax;
        out[b].bot = H - y1 < rmax ? H - y1 : rmax;
    }
    return nb;
}

// floats of one frame's band buffers: radiance + importance with halos, blend + out without
size_t host_frame_floats(int H, int W, int M, int rmax) {
    HostBand bb[HOST_MAX_BANDS];
    const int nb = host_bands(H, rmax, bb);
    size_t f = 0;
    for (int b = 0; b < nb; ++b) {
        const size_t buf = (size_t)(bb[b].top + bb[b].rows + bb[b].bot) * W;
        f += buf * (3 + M) + (size_t)bb[b].rows * W * (M + 3);
        f = (f + 31) & ~(size_t)31;  // keep every band 128-byte aligned
    }
    return f;
}

struct HostStreams {
    cudaStream_t h2d = nullptr, comp = nullptr, d2h = nullptr;
    cudaEvent_t join = nullptr, done = nullptr;
    // workspace carve of the last call (cross-call reuse of the band buffers)
    const void* last_ws = nullptr;
    int last_N = -1, last_H = -1, last_W = -1, last_M = -1, last_rmax = -1, last_in16 = -1;
    cudaEvent_t in[2][HOST_MAX_BANDS] = {}, kern[2][HOST_MAX_BANDS] = {}, out[2][HOST_MAX_BANDS] = {};
    bool ok = false;
    int dev = -1;
};
thread_local HostStreams g_hs;

cudaError_t host_streams(HostStreams** hs) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (!g_hs.ok || g_hs.dev != dev) {
        HostStreams h;
        const unsigned fl = cudaStreamNonBlocking;
        if ((e = cudaStreamCreateWithFlags(&h.h2d, fl)) != cudaSuccess) return e;
        if ((e = cudaStreamCreateWithFlags(&h.comp, fl)) != cudaSuccess) return e;
        if ((e = cudaStreamCreateWithFlags(&h.d2h, fl)) != cudaSuccess) return e;
        const unsigned ef = cudaEventDisableTiming;
        if ((e = cudaEventCreateWithFlags(&h.join, ef)) != cudaSuccess) return e;
        if ((e = cudaEventCreateWithFlags(&h.done, ef)) != cudaSuccess) return e;
        for (int s = 0; s < 2; ++s)
            for (int b = 0; b < HOST_MAX_BANDS; ++b) {
                if ((e = cudaEventCreateWithFlags(&h.in[s][b], ef)) != cudaSuccess) return e;
                if ((e = cudaEventCreateWithFlags(&h.kern[s][b], ef)) != cudaSuccess) return e;
                if ((e = cudaEventCreateWithFlags(&h.out[s][b], ef)) != cudaSuccess) return e;
            }
        h.ok = true;
        h.dev = dev;
        g_hs = h;  // (streams of a previous device are left to the driver at exit)
    }
    *hs = &g_hs;
    return cudaSuccess;
}

// rows [r0, r0+nr) of `planes` planes of an [planes][H][W] host tensor <-> a
// dense [planes][nr][W] device buffer, one 3-D copy
cudaError_t copy_rows(void* dev, const void* host, int W, int H, int planes, int r0, int nr, bool to_dev,
                      cudaStream_t st, size_t esz = sizeof(float)) {
    cudaMemcpy3DParms c = {};
    const size_t pitch = (size_t)W * esz;
    cudaPitchedPtr hp = make_cudaPitchedPtr((void*)((const char*)host + (size_t)r0 * pitch), pitch, W, H);
    cudaPitchedPtr dp = make_cudaPitchedPtr(dev, pitch, W, nr);
    if (to_dev) {
        c.srcPtr = hp;
        c.dstPtr = dp;
        c.kind = cudaMemcpyHostToDevice;
    } else {
        c.srcPtr = dp;
        c.dstPtr = hp;
        c.kind = cudaMemcpyDeviceToHost;
    }
    c.extent = make_cudaExtent(pitch, nr, planes);
    return cudaMemcpy3DAsync(&c, st);
}

}  // namespace

extern "C" {

size_t kmd_host_workspace_bytes(int32_t N, int32_t H, int32_t W, const kmd_config* cfg) {
    if (!cfg || N < 1 || H < 1 || W < 1 || cfg->num_sizes < 1 || cfg->num_sizes > KMD_MAX_SIZES) return 0;
    const size_t frame = host_frame_floats(H, W, cfg->num_sizes, rmax_of(cfg)) * sizeof(float);
    return frame * (N > 1 ? 2 : 1);  // two frames in flight when N > 1
}

}  // extern "C"

namespace {
// the host entry points (fp32 or bf16 importance / logits in host memory)
kmd_status host_entry(const float* radiance_host, const void* importance_host, const void* blend_host,
                      float* out_host, int32_t N, int32_t H, int32_t W, const kmd_config* cfg,
                      void* device_workspace, size_t workspace_bytes, kmd_stream_t stream, int in16) {
    g_err[0] = 0;
    if (N < 0) return fail(KMD_ERR_DIM, "N=%d < 0", N);
    if (N > 0 && (H < 1 || W < 1)) return fail(KMD_ERR_DIM, "H=%d, W=%d must be >= 1", H, W);
    if (!cfg) return fail(KMD_ERR_NULL, "cfg is NULL");
    if (N > 0) {
        kmd_status s = check_cfg(cfg, H, W);
        if (s) return s;
    }
    if (N == 0) return KMD_OK;
    if (!radiance_host || !importance_host || !out_host || !device_workspace)
        return fail(KMD_ERR_NULL, "a host buffer or the workspace is NULL");
    if (cfg->num_sizes > 1 && !blend_host) return fail(KMD_ERR_NULL, "blend is NULL with M=%d > 1", cfg->num_sizes);
    if (in16) {
        if (W % 8 != 0) return fail(KMD_ERR_ALIGN, "bf16 path needs W %% 8 == 0 (W=%d)", W);
        for (int k = 0; k < cfg->num_sizes; ++k)
            if ((cfg->sizes[k] - 1) / 2 > 6)
                return fail(KMD_ERR_CONFIG, "bf16 path supports sizes <= 13 (sizes[%d]=%d)", k, cfg->sizes[k]);
        if ((uintptr_t)device_workspace & 15) return fail(KMD_ERR_ALIGN, "bf16 path needs a 16-byte aligned workspace");
    }
    const size_t esz = in16 ? 2 : 4;
    const size_t need = kmd_host_workspace_bytes(N, H, W, cfg);
    if (workspace_bytes < need)
        return fail(KMD_ERR_DIM, "workspace %zu bytes < required %zu", workspace_bytes, need);
    HostStreams* hs = nullptr;
    cudaError_t e = host_streams(&hs);
    if (e != cudaSuccess) return cuda_fail(e, "host pipeline streams");
    const int M = cfg->num_sizes, rmax = rmax_of(cfg);
    const size_t plane = (size_t)H * W;
    const size_t frame_floats = host_frame_floats(H, W, M, rmax);
    HostBand bb[HOST_MAX_BANDS];
    const int nb = host_bands(H, rmax, bb);
    cudaStream_t user = (cudaStream_t)stream;
    // the kernels and the D2H copies come after everything already queued on
    // the caller's stream.  The H2D copies (host inputs into the workspace) wait
    // only for the workspace: when this call carves it as the previous call on
    // this thread did, band b's buffers wait for that call's band b D2H, so the
    // copies of consecutive calls stream back to back; otherwise for the whole
    // previous call
    if ((e = cudaEventRecord(hs->join, user)) != cudaSuccess) return cuda_fail(e, "event record");
    for (cudaStream_t st : {hs->comp, hs->d2h})
        if ((e = cudaStreamWaitEvent(st, hs->join, 0)) != cudaSuccess) return cuda_fail(e, "stream wait");
    const bool same_carve = hs->last_ws == device_workspace && hs->last_N == N && hs->last_H == H &&
                            hs->last_W == W && hs->last_M == M && hs->last_rmax == rmax && hs->last_in16 == in16;
    if (!same_carve && (e = cudaStreamWaitEvent(hs->h2d, hs->done, 0)) != cudaSuccess)
        return cuda_fail(e, "stream wait");
    hs->last_ws = device_workspace; hs->last_N = N; hs->last_H = H; hs->last_W = W; hs->last_M = M;
    hs->last_rmax = rmax;
    hs->last_in16 = in16;
    for (int n = 0; n < N; ++n) {
        const int set = n & 1;
        float* base = (float*)device_workspace + (size_t)(N > 1 ? set : 0) * frame_floats;
        const float* rh = radiance_host + (size_t)n * 3 * plane;
        const char* ih = (const char*)importance_host + (size_t)n * M * plane * esz;
        const char* bh = M > 1 ? (const char*)blend_host + (size_t)n * M * plane * esz : nullptr;
        float* oh = out_host + (size_t)n * 3 * plane;
        float* cur = base;
        for (int b = 0; b < nb; ++b) {
            const HostBand& B = bb[b];
            const int buf_rows = B.top + B.rows + B.bot;
            float* d_rad = cur;
            float* d_imp = d_rad + (size_t)3 * buf_rows * W;
            float* d_bl = d_imp + (size_t)M * buf_rows * W;
            float* d_out = d_bl + (size_t)M * B.rows * W;
            cur = d_out + (size_t)3 * B.rows * W;
            cur = base + ((size_t)(cur - base) + 31 & ~(size_t)31);
            // the buffers of this set were last used two frames ago (or by the
            // previous call with the same carve): wait for that D2H
            if ((n >= 2 || (n < 2 && same_carve)) &&
                (e = cudaStreamWaitEvent(hs->h2d, hs->out[set][b], 0)) != cudaSuccess)
                return cuda_fail(e, "stream wait");
            const int r0 = B.y0 - B.top;
            if ((e = copy_rows(d_rad, rh, W, H, 3, r0, buf_rows, true, hs->h2d)) != cudaSuccess ||
                (e = copy_rows(d_imp, ih, W, H, M, r0, buf_rows, true, hs->h2d, esz)) != cudaSuccess ||
                (bh && (e = copy_rows(d_bl, bh, W, H, M, B.y0, B.rows, true, hs->h2d, esz)) != cudaSuccess))
                return cuda_fail(e, "H2D band copy");
            if ((e = cudaEventRecord(hs->in[set][b], hs->h2d)) != cudaSuccess) return cuda_fail(e, "event record");
            if ((e = cudaStreamWaitEvent(hs->comp, hs->in[set][b], 0)) != cudaSuccess) return cuda_fail(e, "stream wait");
            kmd::FusedParams bp{};
            bool skip = false;
            kmd_status s = band_params(d_rad, d_imp, bh ? d_bl : nullptr, d_out, 1, B.rows, W, B.top, B.bot, B.y0, H,
                                       cfg, &bp, &skip, in16);
            if (!s && !skip) s = run_fused(bp, cfg, hs->comp);
            if (s) return s;
            if ((e = cudaEventRecord(hs->kern[set][b], hs->comp)) != cudaSuccess) return cuda_fail(e, "event record");
            if ((e = cudaStreamWaitEvent(hs->d2h, hs->kern[set][b], 0)) != cudaSuccess) return cuda_fail(e, "stream wait");
            if ((e = copy_rows(d_out, oh, W, H, 3, B.y0, B.rows, false, hs->d2h)) != cudaSuccess)
                return cuda_fail(e, "D2H band copy");
            if ((e = cudaEventRecord(hs->out[set][b], hs->d2h)) != cudaSuccess) return cuda_fail(e, "event record");
        }
    }
    // the caller's stream resumes after the last band's D2H (d2h is in order)
    if ((e = cudaEventRecord(hs->done, hs->d2h)) != cudaSuccess) return cuda_fail(e, "event record");
    if ((e = cudaStreamWaitEvent(user, hs->done, 0)) != cudaSuccess) return cuda_fail(e, "stream wait");
    return KMD_OK;
}
}  // namespace

extern "C" {

kmd_status kmd_decode_filter_fuse_host(const float* radiance_host, const float* importance_host,
                                       const float* blend_host, float* out_host, int32_t N,
                                       int32_t H, int32_t W, const kmd_config* cfg,
                                       void* device_workspace, size_t workspace_bytes,
                                       kmd_stream_t stream) {
    return host_entry(radiance_host, importance_host, blend_host, out_host, N, H, W, cfg, device_workspace,
                      workspace_bytes, stream, 0);
}

kmd_status kmd_decode_filter_fuse_host_bf16(const float* radiance_host, const uint16_t* importance_host,
                                            const uint16_t* blend_host, float* out_host, int32_t N,
                                            int32_t H, int32_t W, const kmd_config* cfg,
                                            void* device_workspace, size_t workspace_bytes,
                                            kmd_stream_t stream) {
    return host_entry(radiance_host, importance_host, blend_host, out_host, N, H, W, cfg, device_workspace,
                      workspace_bytes, stream, 1);
}

// ---------------------------------------------------------------------------
// NEXT row 2: multi-resolution reconstruction (Eq. 7)
struct MrStreams {
    cudaStream_t aux = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
    int dev = -1;
};
thread_local MrStreams g_ms;
static cudaError_t mr_streams(MrStreams** out) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (g_ms.dev != dev) {
        if ((e = cudaStreamCreateWithFlags(&g_ms.aux, cudaStreamNonBlocking)) != cudaSuccess) return e;
        if ((e = cudaEventCreateWithFlags(&g_ms.fork, cudaEventDisableTiming)) != cudaSuccess) return e;
        if ((e = cudaEventCreateWithFlags(&g_ms.join, cudaEventDisableTiming)) != cudaSuccess) return e;
        g_ms.dev = dev;
    }
    *out = &g_ms;
    return cudaSuccess;
}
static size_t mr_level_floats(int N, int H, int W, int l) {
    return (size_t)N * 3 * (size_t)(H >> l) * (size_t)(W >> l);
}

size_t kmd_mr_workspace_bytes(int32_t N, int32_t H, int32_t W, const kmd_mr_config* cfg) {
    if (!cfg || cfg->levels < 1 || cfg->levels > KMD_MR_MAX_LEVELS || N < 1 || H < 1 || W < 1) return 0;
    // r_l (l >= 1), f_l (all l), c_l (1 <= l < levels-1), each rounded to 32 floats
    size_t f = 0;
    for (int l = 0; l < cfg->levels; ++l) {
        const size_t n = (mr_level_floats(N, H, W, l) + 31) & ~(size_t)31;
        f += n;                                    // f_l
        if (l >= 1) f += n;                        // r_l
        if (l >= 1 && l < cfg->levels - 1) f += n; // c_l
    }
    return f * sizeof(float);
}

kmd_status kmd_downsample2x2(const float* in, float* out, int32_t N, int32_t C, int32_t H, int32_t W,
                             kmd_stream_t stream) {
    g_err[0] = 0;
    if (N < 0 || C < 0) return fail(KMD_ERR_DIM, "N=%d, C=%d must be >= 0", N, C);
    if (N == 0 || C == 0) return KMD_OK;
    if (H < 2 || W < 2 || (H & 1) || (W & 1)) return fail(KMD_ERR_DIM, "H=%d, W=%d must be even and >= 2", H, W);
    if (!in || !out) return fail(KMD_ERR_NULL, "NULL buffer");
    const size_t ib = (size_t)N * C * H * W * sizeof(float);
    if (overlaps(out, ib / 4, in, ib)) return fail(KMD_ERR_ALIAS, "out overlaps in");
    cudaError_t e = kmd::launch_down2(in, out, (long long)N * C, H / 2, W / 2, (cudaStream_t)stream);
    return e == cudaSuccess ? KMD_OK : cuda_fail(e, "downsample launch");
}

kmd_status kmd_combine_resolutions(const float* fine, const float* coarse, const float* alpha, float* out,
                                   int32_t N, int32_t H, int32_t W, kmd_stream_t stream) {
    g_err[0] = 0;
    if (N < 0) return fail(KMD_ERR_DIM, "N=%d < 0", N);
    if (N == 0) return KMD_OK;
    if (H < 2 || W < 2 || (H & 1) || (W & 1)) return fail(KMD_ERR_DIM, "H=%d, W=%d must be even and >= 2", H, W);
    if (!fine || !coarse || !alpha || !out) return fail(KMD_ERR_NULL, "NULL buffer");
    const size_t fb = (size_t)N * 3 * H * W * sizeof(float);
    if (overlaps(out, fb, fine, fb) || overlaps(out, fb, coarse, fb / 4) || overlaps(out, fb, alpha, fb / 3))
        return fail(KMD_ERR_ALIAS, "out overlaps an input");
    cudaError_t e = kmd::launch_combine(fine, coarse, alpha, out, N, H, W, (cudaStream_t)stream);
    return e == cudaSuccess ? KMD_OK : cuda_fail(e, "combine launch");
}

kmd_status kmd_mr_decode_filter_fuse(const float* radiance, const float* const* importance,
                                     const float* const* blend, const float* const* alpha, float* out,
                                     int32_t N, int32_t H, int32_t W, const kmd_mr_config* cfg,
                                     void* workspace, size_t workspace_bytes, kmd_stream_t stream) {
    g_err[0] = 0;
    if (!cfg) return fail(KMD_ERR_NULL, "cfg is NULL");
    const int L = cfg->levels;
    if (L < 1 || L > KMD_MR_MAX_LEVELS) return fail(KMD_ERR_CONFIG, "levels=%d not in [1,%d]", L, KMD_MR_MAX_LEVELS);
    if (N < 0) return fail(KMD_ERR_DIM, "N=%d < 0", N);
    if (N == 0) return KMD_OK;
    const int mask = (1 << (L - 1)) - 1;
    if (H < 1 || W < 1 || (H & mask) || (W & mask))
        return fail(KMD_ERR_DIM, "H=%d, W=%d must be divisible by 2^(levels-1)=%d", H, W, mask + 1);
    for (int l = 0; l < L; ++l) {
        kmd_status s = check_cfg(&cfg->level[l], H >> l, W >> l);
        if (s) return s;
    }
    if (!radiance || !importance || !out || !workspace || (L > 1 && !alpha))
        return fail(KMD_ERR_NULL, "NULL argument");
    for (int l = 0; l < L; ++l) {
        if (!importance[l]) return fail(KMD_ERR_NULL, "importance[%d] is NULL", l);
        if (cfg->level[l].num_sizes > 1 && (!blend || !blend[l])) return fail(KMD_ERR_NULL, "blend[%d] is NULL", l);
        if (l < L - 1 && !alpha[l]) return fail(KMD_ERR_NULL, "alpha[%d] is NULL", l);
    }
    if (workspace_bytes < kmd_mr_workspace_bytes(N, H, W, cfg))
        return fail(KMD_ERR_DIM, "workspace %zu bytes < required %zu", workspace_bytes,
                    kmd_mr_workspace_bytes(N, H, W, cfg));
    cudaStream_t st = (cudaStream_t)stream;
    // carve the workspace: for each level l: f_l, r_l (l>=1), c_l (1<=l<L-1)
    float* ws = (float*)workspace;
    float *r[KMD_MR_MAX_LEVELS] = {}, *f[KMD_MR_MAX_LEVELS] = {}, *c[KMD_MR_MAX_LEVELS] = {};
    for (int l = 0; l < L; ++l) {
        const size_t n = (mr_level_floats(N, H, W, l) + 31) & ~(size_t)31;
        f[l] = ws; ws += n;
        if (l >= 1) { r[l] = ws; ws += n; }
        if (l >= 1 && l < L - 1) { c[l] = ws; ws += n; }
    }
    r[0] = const_cast<float*>(radiance);
    cudaError_t e;
    int l0 = 1;
    if (L >= 3) {  // levels 1 and 2 in one pass over the frame
        if ((e = kmd::launch_down4(r[0], r[1], r[2], N * 3, H >> 2, W >> 2, st)) != cudaSuccess)
            return cuda_fail(e, "downsample launch");
        l0 = 3;
    }
    for (int l = l0; l < L; ++l)
        if ((e = kmd::launch_down2(r[l - 1], r[l], (long long)N * 3, H >> l, W >> l, st)) != cudaSuccess)
            return cuda_fail(e, "downsample launch");
    if (L == 1) return kmd_decode_filter_fuse(r[0], importance[0], blend ? blend[0] : nullptr, out, N, H, W,
                                              &cfg->level[0], stream);
    // Fused path (the paper's configuration: every level M = 2 sizes <= 13 with
    // fusion logits, TMA-compatible widths and alignment): from the coarsest
    // level up, each level's kernel applies Eq. 7 with the level below in its
    // epilogue (28-row tiles, kmd_tma_mr.cu), so no fine-level filtered image
    // makes a round trip through HBM and no separate combine runs.
    {
        bool fused = true;
        uintptr_t amask = (uintptr_t)out;
        for (int l = 0; l < L && fused; ++l) {
            const kmd_config& lc = cfg->level[l];
            fused = lc.num_sizes == 2 && lc.blend_is_logits && blend && blend[l] && ((W >> l) % 4) == 0 &&
                    (l == L - 1 || (((H >> l) % 2) == 0 && ((W >> l) % 2) == 0));
            for (int i = 0; i < lc.num_sizes && fused; ++i) fused = lc.sizes[i] <= 13;
            if (fused) amask |= (uintptr_t)r[l] | (uintptr_t)importance[l] | (uintptr_t)blend[l] | (uintptr_t)f[l] |
                                (l < L - 1 ? (uintptr_t)alpha[l] : 0);
        }
        if (fused && (amask & 15) == 0) {
            for (int l = L - 1; l >= 0; --l) {
                kmd::FusedParams p{};
                p.rad = r[l]; p.imp = importance[l]; p.blend = blend[l];
                p.out = l == 0 ? out : f[l];
                p.N = N; p.W = W >> l; p.H = H >> l;
                p.row_base = 0; p.buf_rows = p.H; p.out_y0 = 0; p.out_rows = p.H;
                const kmd_config& lc = cfg->level[l];
                p.M = lc.num_sizes; p.rmax = rmax_of(&lc); p.blend_is_logits = lc.blend_is_logits;
                p.debug = debug_env();
                for (int i = 0; i < KMD_MAX_SIZES; ++i) p.sizes[i] = i < lc.num_sizes ? lc.sizes[i] : 1;
                if (l < L - 1) {
                    p.cmb_coarse = f[l + 1];  // the combined next-coarser level (the coarsest: as filtered)
                    p.cmb_alpha = alpha[l];
                }
                if ((e = kmd::launch_fused_tma_mr(p, st)) != cudaSuccess) return cuda_fail(e, "MR level launch");
            }
            return KMD_OK;
        }
    }
    // The coarse levels (and their Eq. 7 combines) run on an auxiliary stream,
    // concurrently with level 0, each persistent launch on its share of the SMs
    // (proportional to its tiles): the small levels no longer run alone.
    MrStreams* ms = nullptr;
    if ((e = mr_streams(&ms)) != cudaSuccess) return cuda_fail(e, "multi-resolution streams");
    int sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    long long t0 = 0, t12 = 0;
    for (int l = 0; l < L; ++l) {
        const long long t = (long long)N * (((W >> l) + 51) / 52) * (((H >> l) + 26) / 27);
        (l == 0 ? t0 : t12) += t;
    }
    int cap0 = (int)((double)sms * (double)t0 / (double)(t0 + t12) + 0.5);
    cap0 = cap0 < 1 ? 1 : (cap0 > sms - 1 ? sms - 1 : cap0);
    if ((e = cudaEventRecord(ms->fork, st)) != cudaSuccess) return cuda_fail(e, "event record");
    if ((e = cudaStreamWaitEvent(ms->aux, ms->fork, 0)) != cudaSuccess) return cuda_fail(e, "stream wait");
    struct CapGuard {
        ~CapGuard() { g_max_ctas = 0; }
    } guard;
    g_max_ctas = sms - cap0;
    for (int l = 1; l < L; ++l) {
        kmd_status s = kmd_decode_filter_fuse(r[l], importance[l], blend ? blend[l] : nullptr, f[l], N, H >> l,
                                              W >> l, &cfg->level[l], ms->aux);
        if (s) return s;
    }
    // Eq. 7 from the coarsest level: c_{L-1} = f_{L-1}; c_l = combine(f_l, c_{l+1}, alpha_l)
    const float* coarse = f[L - 1];
    for (int l = L - 2; l >= 1; --l) {
        if ((e = kmd::launch_combine(f[l], coarse, alpha[l], c[l], N, H >> l, W >> l, ms->aux)) != cudaSuccess)
            return cuda_fail(e, "combine launch");
        coarse = c[l];
    }
    if ((e = cudaEventRecord(ms->join, ms->aux)) != cudaSuccess) return cuda_fail(e, "event record");
    g_max_ctas = cap0;
    kmd_status s0 = kmd_decode_filter_fuse(r[0], importance[0], blend ? blend[0] : nullptr, f[0], N, H, W,
                                           &cfg->level[0], stream);
    if (s0) return s0;
    g_max_ctas = 0;
    if ((e = cudaStreamWaitEvent(st, ms->join, 0)) != cudaSuccess) return cuda_fail(e, "stream wait");
    if ((e = kmd::launch_combine(f[0], coarse, alpha[0], out, N, H, W, st)) != cudaSuccess)
        return cuda_fail(e, "combine launch");
    return KMD_OK;
}

// ---------------------------------------------------------------------------
// NEXT row 3: backward
size_t kmd_backward_workspace_bytes(int32_t N, int32_t H, int32_t W, const kmd_config* cfg) {
    if (!cfg || N < 1 || H < 1 || W < 1 || cfg->num_sizes < 1 || cfg->num_sizes > KMD_MAX_SIZES) return 0;
    // the h_i field of the TMA path (pass A -> pass B); the one-launch fallback needs none
    return kmd::bwd_tma_workspace_bytes(N, H, W, cfg->num_sizes);
}

kmd_status kmd_decode_filter_fuse_backward(const float* radiance, const float* importance, const float* blend,
                                           const float* grad_out, float* grad_importance, float* grad_blend,
                                           int32_t N, int32_t H, int32_t W, const kmd_config* cfg,
                                           void* workspace, size_t workspace_bytes, kmd_stream_t stream) {
    g_err[0] = 0;
    if (N < 0) return fail(KMD_ERR_DIM, "N=%d < 0", N);
    if (N > 0 && (H < 1 || W < 1)) return fail(KMD_ERR_DIM, "H=%d, W=%d must be >= 1", H, W);
    if (!cfg) return fail(KMD_ERR_NULL, "cfg is NULL");
    if (N > 0) {
        kmd_status s = check_cfg(cfg, H, W);
        if (s) return s;
    }
    if (N == 0) return KMD_OK;
    if (!radiance || !importance || !grad_out || !grad_importance) return fail(KMD_ERR_NULL, "NULL argument");
    if (cfg->num_sizes > 1 && !blend) return fail(KMD_ERR_NULL, "blend is NULL with M=%d > 1", cfg->num_sizes);
    if (workspace_bytes < kmd_backward_workspace_bytes(N, H, W, cfg))
        return fail(KMD_ERR_DIM, "workspace too small");
    for (int i = 0; i < cfg->num_sizes; ++i)
        if (cfg->sizes[i] > 13)
            return fail(KMD_ERR_CONFIG, "backward: sizes[%d]=%d > 13 (both backward kernels stage r_max <= 6 halos)",
                        i, cfg->sizes[i]);
    const int M = cfg->num_sizes;
    cudaError_t e;
    // the TMA path stores dL/dI through a tensor map: grad_importance must be
    // 16-byte aligned as well (else the one-launch kernel runs)
    if (workspace && kmd::bwd_tma_supported(H, W, M, cfg->sizes, radiance, importance, grad_out, workspace) &&
        ((uintptr_t)grad_importance & 15) == 0 && (M == 1 || ((uintptr_t)blend & 15) == 0)) {
        kmd::set_last_kernel(kmd::LK_BWD_TMA);
        e = kmd::launch_backward_tma(radiance, importance, M > 1 ? blend : nullptr, grad_out, grad_importance,
                                     grad_blend, N, H, W, M, cfg->sizes, cfg->blend_is_logits, workspace,
                                     (cudaStream_t)stream);
    } else {
        kmd::set_last_kernel(kmd::LK_BWD_TILE);
        e = kmd::launch_backward(radiance, importance, M > 1 ? blend : nullptr, grad_out, grad_importance,
                                 grad_blend, N, H, W, M, cfg->sizes, cfg->blend_is_logits, (float*)workspace,
                                 (cudaStream_t)stream);
    }
    return e == cudaSuccess ? KMD_OK : cuda_fail(e, "backward launch");
}

// ---------------------------------------------------------------------------
// NEXT row 4: temporal accumulation
kmd_status kmd_temporal_accumulate(const float* cur_radiance, const float* prev_radiance,
                                   const float* prev_position, const float* prev_normal,
                                   const uint8_t* prev_valid, const float* cur_position,
                                   const float* cur_normal, const float* motion, float* accum,
                                   uint8_t* mask, int32_t N, int32_t H, int32_t W, float pos_tol,
                                   float normal_tol, float alpha, kmd_stream_t stream) {
    g_err[0] = 0;
    if (N < 0 || (N > 0 && (H < 1 || W < 1))) return fail(KMD_ERR_DIM, "bad N/H/W");
    if (!(pos_tol > 0.f)) return fail(KMD_ERR_CONFIG, "pos_tol must be > 0");
    if (!(normal_tol > 0.f && normal_tol <= 1.f)) return fail(KMD_ERR_CONFIG, "normal_tol must be in (0, 1]");
    if (!(alpha > 0.f && alpha <= 1.f)) return fail(KMD_ERR_CONFIG, "alpha must be in (0, 1]");
    if (N == 0) return KMD_OK;
    if (!cur_radiance || !prev_radiance || !prev_position || !prev_normal || !prev_valid || !cur_position ||
        !cur_normal || !motion || !accum)
        return fail(KMD_ERR_NULL, "NULL buffer");
    const size_t b3 = (size_t)N * 3 * H * W * sizeof(float), b1 = (size_t)N * H * W;
    if (overlaps(accum, b3, prev_radiance, b3) || overlaps(accum, b3, prev_position, b3) ||
        overlaps(accum, b3, prev_normal, b3) || overlaps(accum, b3, prev_valid, b1) ||
        (mask && (overlaps(mask, b1, prev_radiance, b3) || overlaps(mask, b1, prev_valid, b1) ||
                  overlaps(mask, b1, accum, b3))))
        return fail(KMD_ERR_ALIAS, "accum / mask overlap a previous-frame buffer");
    cudaError_t e = kmd::launch_temporal(cur_radiance, prev_radiance, prev_position, prev_normal, prev_valid,
                                         cur_position, cur_normal, motion, accum, mask, N, H, W, pos_tol,
                                         normal_tol, alpha, (cudaStream_t)stream);
    return e == cudaSuccess ? KMD_OK : cuda_fail(e, "temporal launch");
}

int64_t kmd_algorithmic_bytes(int32_t N, int32_t H, int32_t W, const kmd_config* cfg,
                              int32_t has_blend) {
    if (!cfg || N < 0 || H < 0 || W < 0) return -1;
    const int64_t M = cfg->num_sizes;
    return (int64_t)N * H * W * 4 * (3 + M + (has_blend ? M : 0) + 3);
}

int32_t kmd_launches_per_call(void) { return 1; }

const char* kmd_status_string(kmd_status s) {
    switch (s) {
        case KMD_OK: return "KMD_OK";
        case KMD_ERR_NULL: return "KMD_ERR_NULL";
        case KMD_ERR_CONFIG: return "KMD_ERR_CONFIG";
        case KMD_ERR_DIM: return "KMD_ERR_DIM";
        case KMD_ERR_ALIGN: return "KMD_ERR_ALIGN";
        case KMD_ERR_ALIAS: return "KMD_ERR_ALIAS";
        case KMD_ERR_CUDA: return "KMD_ERR_CUDA";
        case KMD_ERR_NCCL: return "KMD_ERR_NCCL";
    }
    return "KMD_ERR_UNKNOWN";
}

const char* kmd_last_error(void) { return g_err; }

int32_t kmd_version(void) { return KMD_VERSION_MAJOR * 100 + KMD_VERSION_MINOR; }

int32_t kmd_last_kernel(void) { return g_last_kernel; }

}  // extern "C"
