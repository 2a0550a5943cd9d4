// kmd_ws.cu -- v2 fused decode + filter + fuse: persistent, warp-specialised
// producer/consumer kernel for sm_100a (kernel sizes k <= 13, M <= 8).
//
// Arithmetic.  Eq. 3's weight of q is exp(I(q)) for every
// window containing q (the paper's "weight sharing"), so
// Eq. 3 + Eq. 4 are exactly a ratio of two k x k box sums of the premultiplied
// field P = (e, e r, e g, e b), e = exp(I):
//     R^k(p) = box_k(e r)(p) / box_k(e)(p).
// The box sums are separable and add-only (no subtraction, so no cancellation
// for any dynamic range of e).
//
// Work decomposition.  Output tile = 52 columns x 32 rows of one frame; the
// field of every size is evaluated on the same 64 columns [x0-6, x0+58), so a
// (size, 32-column half) job is one full warp with a warp-uniform window radius.
//   * 6 producer warps: job = (tile, size i, half).  Each lane owns one field
//     column: loads I_i and r,g,b down the column (coalesced across lanes),
//     e = expf(I) once per field pixel, vertical k-tap sums in registers
//     (shared-core grouping, fixed order), writes the 32 vertical sums V and the
//     blend logits of its columns into a shared-memory slot.
//   * 4 consumer warps: thread = (row, 13-pixel segment).  Per size, reads 13+2R
//     vertical sums, horizontal k-tap sums in registers, R = num * rcp(den), and
//     folds it into an online softmax over the blend logits (Eq. 5 with
//     alpha = softmax(B)).  After the last size the tile
//     is staged in shared memory and written out coalesced.
//   * A ring of 4 slots with mbarrier full/empty pairs couples the two roles.
// Tiles are aligned to a global 52 x 32 grid and every sum is taken in a
// fixed order, so results depend on the output pixel only (bitwise-equal row
// bands).  A (tile, size) whose importance leaves [KMD_EXP_SAFE_LO,
// KMD_EXP_SAFE_HI] (or radiance beyond KMD_RADIANCE_SAFE) is recomputed by the
// consumers with a per-window max shift (R2/R13).
#include "kmd_common.cuh"
#include "kmd_kernels.h"

namespace kmd {
namespace ws {

constexpr int RMAX = 6;
constexpr int TW = 52;            // output columns per tile
constexpr int TH = 32;            // output rows per tile
constexpr int SEG = 13;           // output pixels per consumer thread (TW / 4)
constexpr int NSLOT = 4;
constexpr int NPROD = 6;          // producer warps
constexpr int NCONS = 4;          // consumer warps
constexpr int NTHREADS = (NPROD + NCONS) * 32;
constexpr int VS = 68;            // V / Bs row stride (== 4 mod 8: conflict-free consumer reads)
constexpr float L2E = 1.4426950408889634f;

struct Smem {
    float4 V[NSLOT][TH][VS];      // vertical box sums of (e, e r, e g, e b)
    float Bs[NSLOT][TH][VS];      // blend logits (or alphas) of size i at the tile pixels
    float stage[3][TH][TW];       // output tile staging for coalesced stores
    unsigned long long full[NSLOT];
    unsigned long long empty[NSLOT];
    int flags[NSLOT][2];
};

__device__ __forceinline__ void consumer_bar() { asm volatile("bar.sync 1, %0;" ::"n"(NCONS * 32) : "memory"); }

// Window sums out[x] = sum_{j=x}^{x+2R} P[j] for the group x in [G0, G0+GS),
// GS <= 2R+1: every window of the group contains the shared core
// P[G0+GS-1 .. G0+2R]; the left parts are suffix sums of P[G0 .. G0+GS-2] and
// the right parts prefix sums of P[G0+2R+1 .. G0+GS-1+2R].  2R + 3 GS - 5
// adds per group, all of non-negative terms, in an order fixed by (R, G0, GS).
// All indices are compile-time constants so P stays in registers.
template <int R, int G0, int GS, int NP, class Emit>
__device__ __forceinline__ void group_sums_n(const float4 (&P)[NP], Emit&& emit) {
    static_assert(GS >= 1 && GS <= 2 * R + 1, "group wider than the window");
    static_assert(G0 + GS - 1 + 2 * R < NP, "window beyond the field line");
    float4 core = P[G0 + GS - 1];
#pragma unroll
    for (int j = G0 + GS; j <= G0 + 2 * R; ++j) core = add4(core, P[j]);
    if constexpr (GS == 1) {
        emit(G0, core);
    } else {
        float4 suf[GS - 1];
        suf[GS - 2] = P[G0 + GS - 2];
#pragma unroll
        for (int k = GS - 3; k >= 0; --k) suf[k] = add4(P[G0 + k], suf[k + 1]);
        emit(G0, add4(suf[0], core));
        float4 pre = P[G0 + 1 + 2 * R];
#pragma unroll
        for (int k = 1; k < GS; ++k) {
            if (k > 1) pre = add4(pre, P[G0 + k + 2 * R]);
            const float4 t = (k == GS - 1) ? core : add4(suf[k], core);
            emit(G0 + k, add4(t, pre));
        }
    }
}

// All N outputs of a line in groups of G (the last one shorter).  Field values
// are produced by `field(j)` right before the first group that needs them.
template <int R, int N, int G, int G0, int NP, class Field, class Emit>
__device__ __forceinline__ void box_line_rec(float4 (&P)[NP], Field& field, Emit& emit) {
    if constexpr (G0 < N) {
        constexpr int GS = (N - G0 < G) ? (N - G0) : G;
        constexpr int F0 = (G0 == 0) ? 0 : G0 + 2 * R;
        constexpr int F1 = G0 + GS + 2 * R;
#pragma unroll
        for (int f = F0; f < F1; ++f) P[f] = field(f);
        group_sums_n<R, G0, GS>(P, emit);
        box_line_rec<R, N, G, G0 + G>(P, field, emit);
    }
}

template <int R, int N, int G, class Field, class Emit>
__device__ __forceinline__ void box_line(Field&& field, Emit&& emit) {
    float4 P[N + 2 * R];
    box_line_rec<R, N, G, 0>(P, field, emit);
}

template <int R> struct VG { static constexpr int value = R == 0 ? 1 : (R <= 2 ? 2 : (R == 3 ? 4 : 8)); };
template <int R> struct HG { static constexpr int value = R == 0 ? 1 : (R <= 2 ? 2 : 7); };

struct TileCoord {
    int n, x0, y0;
};

__device__ __forceinline__ TileCoord tile_of(const FusedParams& p, int t, int tiles_x, int tiles_y) {
    TileCoord c;
    const int per_frame = tiles_x * tiles_y;
    c.n = t / per_frame;
    const int r = t - c.n * per_frame;
    const int ty = r / tiles_x;
    c.x0 = (r - ty * tiles_x) * TW;
    c.y0 = p.tile_y_begin + ty * TH;
    return c;
}

__device__ __forceinline__ int brow(const FusedParams& p, int gy) {
    return clampi(clampi(gy, 0, p.H - 1) - p.row_base, 0, p.buf_rows - 1);
}

// ------------------------------------------------------------------ producer
template <int R>
__device__ __forceinline__ void produce(const FusedParams& p, Smem& sm, int s, int h, const TileCoord& tc, int i,
                                        unsigned empty_parity) {
    const int lane = threadIdx.x & 31;
    const int fc = h * 32 + lane;                         // field column in [0, 64)
    const int gx = clampi(tc.x0 - RMAX + fc, 0, p.W - 1); // reading R1: clamp-to-edge
    const size_t bplane = (size_t)p.buf_rows * p.W;
    const float* Ii = p.imp + ((size_t)tc.n * p.M + i) * bplane + gx;
    const float* rp = p.rad + (size_t)tc.n * 3 * bplane + gx;
    float vmin = INFINITY, vmax = -INFINITY, rabs = 0.f;

    auto field = [&](int f) -> float4 {
        const size_t off = (size_t)brow(p, tc.y0 - R + f) * p.W;
        const float v = __ldg(Ii + off);
        const float r = __ldg(rp + off), g = __ldg(rp + bplane + off), b = __ldg(rp + 2 * bplane + off);
        vmin = fminf(vmin, v);
        vmax = fmaxf(vmax, v);
        rabs = fmaxf(rabs, fmaxf(fabsf(r), fmaxf(fabsf(g), fabsf(b))));
        const float e = expf(v);  // once per field pixel: Eq. 3's shared weight
        const float2 eg = __fmul2_rn(make_float2(e, e), make_float2(r, g));
        return make_float4(e, eg.x, eg.y, e * b);
    };

    // blend logits of this size at the tile pixels (no halo needed)
    const int ox = tc.x0 - RMAX + fc;  // output column of this lane (valid if in [x0, x0+52))
    const bool has_b = p.blend != nullptr && fc >= RMAX && fc < RMAX + TW;
    const size_t oplane = (size_t)p.out_rows * p.W;
    const float* Bi = p.blend ? p.blend + ((size_t)tc.n * p.M + i) * oplane + min(ox, p.W - 1) : nullptr;

    mbar_wait(&sm.empty[s], empty_parity);
    float4* Vcol = &sm.V[s][0][fc];
    box_line<R, TH, VG<R>::value>(field, [&](int oy, float4 v) { Vcol[oy * VS] = v; });
    if (has_b) {
#pragma unroll 4
        for (int oy = 0; oy < TH; ++oy) {
            const int row = clampi(tc.y0 + oy - p.out_y0, 0, p.out_rows - 1);
            sm.Bs[s][oy][fc] = __ldg(Bi + (size_t)row * p.W);
        }
    }
    const bool bad = !(vmin >= KMD_EXP_SAFE_LO && vmax <= KMD_EXP_SAFE_HI) || !(rabs <= KMD_RADIANCE_SAFE);
    const unsigned any = __any_sync(0xffffffffu, bad);
    if (lane == 0) sm.flags[s][h] = any ? 1 : 0;
    __syncwarp();
    mbar_arrive(&sm.full[s]);
}

// ------------------------------------------------------------------ consumer
struct ConsState {
    float m[SEG], S[SEG], acc[SEG][3];
};

__device__ __forceinline__ void fuse_one(const FusedParams& p, ConsState& st, int j, float b, float den, float n0,
                                         float n1, float n2) {
    const float rden = rcp_approx(den);
    if (p.M == 1) {
        st.acc[j][0] = n0 * rden;
        st.acc[j][1] = n1 * rden;
        st.acc[j][2] = n2 * rden;
    } else if (p.blend_is_logits) {
        // online softmax over the M logits (exactly softmax(B) . R at the end)
        const float mn = fmaxf(st.m[j], b);
        const float cold = ex2_approx((st.m[j] - mn) * L2E);
        const float a = ex2_approx((b - mn) * L2E);
        st.m[j] = mn;
        st.S[j] = fmaf(st.S[j], cold, a);
        const float w = a * rden;
        st.acc[j][0] = fmaf(st.acc[j][0], cold, w * n0);
        st.acc[j][1] = fmaf(st.acc[j][1], cold, w * n1);
        st.acc[j][2] = fmaf(st.acc[j][2], cold, w * n2);
    } else {
        const float w = b * rden;
        st.acc[j][0] = fmaf(w, n0, st.acc[j][0]);
        st.acc[j][1] = fmaf(w, n1, st.acc[j][1]);
        st.acc[j][2] = fmaf(w, n2, st.acc[j][2]);
    }
}

template <int R>
__device__ __forceinline__ void consume(const FusedParams& p, Smem& sm, ConsState& st, int s, int ty, int seg) {
    const float4* Vrow = &sm.V[s][ty][SEG * seg + RMAX - R];
    const float* Brow = &sm.Bs[s][ty][SEG * seg + RMAX];
    box_line<R, SEG, HG<R>::value>([&](int j) { return Vrow[j]; },
                                   [&](int x, float4 v) { fuse_one(p, st, x, Brow[x], v.x, v.y, v.z, v.w); });
}

// per-window max-shifted evaluation of one pixel (exact rewrite of Eq. 3,
// reading R2): returns (den, num_r, num_g, num_b)
__device__ __noinline__ float4 fallback_pixel(const FusedParams& p, const TileCoord& tc, int i, int x, int y) {
    const int R = (p.sizes[i] - 1) / 2;
    const size_t bplane = (size_t)p.buf_rows * p.W;
    const float* Ii = p.imp + ((size_t)tc.n * p.M + i) * bplane;
    const float* rp = p.rad + (size_t)tc.n * 3 * bplane;
    x = min(x, p.W - 1);
    float m = -INFINITY;
    for (int dy = -R; dy <= R; ++dy)
        for (int dx = -R; dx <= R; ++dx)
            m = fmaxf(m, __ldg(Ii + (size_t)brow(p, y + dy) * p.W + clampi(x + dx, 0, p.W - 1)));
    float den = 0.f, n0 = 0.f, n1 = 0.f, n2 = 0.f;
    for (int dy = -R; dy <= R; ++dy)
        for (int dx = -R; dx <= R; ++dx) {
            const size_t off = (size_t)brow(p, y + dy) * p.W + clampi(x + dx, 0, p.W - 1);
            const float e = expf(__ldg(Ii + off) - m);
            den += e;
            n0 = fmaf(e, __ldg(rp + off), n0);
            n1 = fmaf(e, __ldg(rp + bplane + off), n1);
            n2 = fmaf(e, __ldg(rp + 2 * bplane + off), n2);
        }
    return make_float4(den, n0, n1, n2);
}

__device__ __forceinline__ void consume_fallback(const FusedParams& p, Smem& sm, ConsState& st, int s, int ty,
                                                 int seg, const TileCoord& tc, int i) {
#pragma unroll
    for (int j = 0; j < SEG; ++j) {
        const float4 v = fallback_pixel(p, tc, i, tc.x0 + SEG * seg + j, tc.y0 + ty);
        fuse_one(p, st, j, sm.Bs[s][ty][SEG * seg + RMAX + j], v.x, v.y, v.z, v.w);
    }
}

// ------------------------------------------------------------------- kernel
__global__ void __launch_bounds__(NTHREADS, 1) fused_ws_kernel(const __grid_constant__ FusedParams p, int tiles_x, int tiles_y, int n_tiles) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
    const int warp = threadIdx.x >> 5;

    if (threadIdx.x == 0) {
        for (int s = 0; s < NSLOT; ++s) {
            mbar_init(&sm.full[s], 2 * 32);       // two producer warps (halves), every lane
            mbar_init(&sm.empty[s], NCONS * 32);  // every consumer thread
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    const int M = p.M;
    if (warp < NPROD) {
        // ---------------- producers: jobs j = warp, warp + NPROD, ... --------
        const int jobs_per_tile = 2 * M;
        for (int j = warp;; j += NPROD) {
            const int tl = j / jobs_per_tile;
            const int t = blockIdx.x + tl * gridDim.x;
            if (t >= n_tiles) break;
            const int rem = j - tl * jobs_per_tile;
            const int i = rem >> 1, h = rem & 1;
            const int seq = tl * M + i;
            const int s = seq % NSLOT;
            const unsigned par = ((seq / NSLOT) & 1) ^ 1;
            const TileCoord tc = tile_of(p, t, tiles_x, tiles_y);
            switch ((p.sizes[i] - 1) / 2) {
                case 0: produce<0>(p, sm, s, h, tc, i, par); break;
                case 1: produce<1>(p, sm, s, h, tc, i, par); break;
                case 2: produce<2>(p, sm, s, h, tc, i, par); break;
                case 3: produce<3>(p, sm, s, h, tc, i, par); break;
                case 4: produce<4>(p, sm, s, h, tc, i, par); break;
                case 5: produce<5>(p, sm, s, h, tc, i, par); break;
                default: produce<6>(p, sm, s, h, tc, i, par); break;
            }
        }
    } else {
        // ---------------- consumers ------------------------------------------
        const int c = threadIdx.x - NPROD * 32;
        const int ty = c >> 2, seg = c & 3;
        const size_t oplane = (size_t)p.out_rows * p.W;
        for (int tl = 0;; ++tl) {
            const int t = blockIdx.x + tl * gridDim.x;
            if (t >= n_tiles) break;
            const TileCoord tc = tile_of(p, t, tiles_x, tiles_y);
            ConsState st;
#pragma unroll
            for (int j = 0; j < SEG; ++j) {
                st.m[j] = -INFINITY;
                st.S[j] = 0.f;
                st.acc[j][0] = st.acc[j][1] = st.acc[j][2] = 0.f;
            }
            for (int i = 0; i < M; ++i) {
                const int seq = tl * M + i;
                const int s = seq % NSLOT;
                mbar_wait(&sm.full[s], (seq / NSLOT) & 1);
                if (sm.flags[s][0] | sm.flags[s][1]) {
                    consume_fallback(p, sm, st, s, ty, seg, tc, i);
                } else {
                    switch ((p.sizes[i] - 1) / 2) {
                        case 0: consume<0>(p, sm, st, s, ty, seg); break;
                        case 1: consume<1>(p, sm, st, s, ty, seg); break;
                        case 2: consume<2>(p, sm, st, s, ty, seg); break;
                        case 3: consume<3>(p, sm, st, s, ty, seg); break;
                        case 4: consume<4>(p, sm, st, s, ty, seg); break;
                        case 5: consume<5>(p, sm, st, s, ty, seg); break;
                        default: consume<6>(p, sm, st, s, ty, seg); break;
                    }
                }
                mbar_arrive(&sm.empty[s]);
            }
            // ---- normalise, stage, store coalesced -----------------------------
            consumer_bar();  // previous tile's stores have read the staging buffer
#pragma unroll
            for (int j = 0; j < SEG; ++j) {
                const float sc = (M > 1 && p.blend_is_logits) ? rcp_approx(st.S[j]) : 1.0f;
                float o0 = st.acc[j][0] * sc, o1 = st.acc[j][1] * sc, o2 = st.acc[j][2] * sc;
                const int gx = tc.x0 + SEG * seg + j, gy = tc.y0 + ty;
                if (gx < p.W && gy >= p.out_y0 && gy < p.out_y0 + p.out_rows) remodulate(p, tc.n, gy, gx, o0, o1, o2);
                sm.stage[0][ty][SEG * seg + j] = o0;
                sm.stage[1][ty][SEG * seg + j] = o1;
                sm.stage[2][ty][SEG * seg + j] = o2;
            }
            consumer_bar();
            float* out = p.out + (size_t)tc.n * 3 * oplane;
            for (int idx = c; idx < 3 * TH * TW; idx += NCONS * 32) {
                const int ch = idx / (TH * TW);
                const int rr = idx - ch * TH * TW;
                const int oy = rr / TW, ox = rr - oy * TW;
                const int gy = tc.y0 + oy, gx = tc.x0 + ox;
                if (gx < p.W && gy >= p.out_y0 && gy < p.out_y0 + p.out_rows)
                    out[ch * oplane + (size_t)(gy - p.out_y0) * p.W + gx] = sm.stage[ch][oy][ox];
            }
        }
    }
}

}  // namespace ws

bool ws_supported(const FusedParams& p) {
    if (p.M < 1 || p.M > KMD_MAX_SIZES) return false;
    for (int i = 0; i < p.M; ++i)
        if ((p.sizes[i] - 1) / 2 > ws::RMAX) return false;
    return true;
}

cudaError_t launch_fused_ws(FusedParams p, cudaStream_t stream) {
    using namespace ws;
    p.tile_y_begin = (p.out_y0 / TH) * TH;
    const int tiles_y = (p.out_y0 + p.out_rows - p.tile_y_begin + TH - 1) / TH;
    const int tiles_x = (p.W + TW - 1) / TW;
    const long long n_tiles = (long long)tiles_x * tiles_y * p.N;
    if (n_tiles > 0x7fffffff) return cudaErrorInvalidValue;
    int dev = 0, sms = 148;
    cudaError_t err = cudaGetDevice(&dev);
    if (err != cudaSuccess) return err;
    err = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (err != cudaSuccess) return err;
    const size_t smem = sizeof(Smem);
    err = cudaFuncSetAttribute(fused_ws_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return err;
    const int grid = (int)(n_tiles < sms ? n_tiles : sms);
    fused_ws_kernel<<<grid, NTHREADS, smem, stream>>>(p, tiles_x, tiles_y, (int)n_tiles);
    return cudaGetLastError();
}

}  // namespace kmd
