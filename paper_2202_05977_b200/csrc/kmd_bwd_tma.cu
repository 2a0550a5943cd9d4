// kmd_bwd_tma.cu -- NEXT row 3, fast path: the backward of the fused decoder
// as three TMA / elementwise passes (Eq. 1: the kernel
// maps are trained end to end through Eq. 3-5).
//
//   pass A (kmd_tma.cu, SpecBwdH): the forward's tiles and box sums; per size i
//          and pixel p the fusion warps stage s_i(p) = a_i / den_i and
//          d_i(p) = G.R_i (a_i = softmax_i(B)(p), G = dL/dRhat(p)) and TMA-store
//          them to the workspace [N*M][2][H][W];
//   pass B (here): T_i = Bt(h_i), h_i = s_i (G, d_i), the transposed
//          clamp-to-edge box: the same warp-specialised pipeline, the field
//          value h_i(q) formed from TMA boxes of (s_i, d_i) and of G (zero
//          outside the frame: TMA's out-of-bounds fill), and the clamped taps folded back
//          onto the border rows (field warps) and columns (fusion warps); the
//          fusion warps finish dL/dI_i(q) = e_i(q) (r(q) . T_i.xyz - T_i.w);
//   pass C (here): dL/dB_i = a_i (G.R_i - sum_j a_j G.R_j), elementwise.
//
// Pass B per CTA (one per SM), per 52 x 27 tile, per size i:
//   warp 0       TMA: the G box [3][39][68] per tile (double-buffered), the
//                (s_i, d_i) box [2][39][68] (2-deep ring) and the I_i
//                box [27][56] of the tile's own pixels (4-deep ring);
//   warps 1-4    field: vertical Gil-Werman sums of h_i per column (+ folds);
//   warps 5-11   fusion: horizontal sums (+ folds), the dL/dI epilogue.
// Unshifted exp: importance in (-80, 80) (header note).
#include <cuda.h>

#include <cstdlib>
#include <mutex>

#include "kmd_common.cuh"
#include "kmd_gw.cuh"
#include "kmd_kernels.h"

namespace kmd {
namespace bwd {

constexpr int RMAX = 6;
constexpr int TW = 52, TH = 27, FH = TH + 2 * RMAX;  // 39 field rows
constexpr int XOFF = 8, BW = 68, VS = 68, BBW = 56;
constexpr int SEG = 7, NSEG = 8;
constexpr int NH = 2, NB = 2, NV = 3;
constexpr int NFIELD = 4, NFUSE = (TH * NSEG + 31) / 32;  // 7
constexpr int NTHREADS = (1 + NFIELD + NFUSE) * 32;

// boxes: rows y0-6 .. y0+32, columns x0-8 .. x0+59, zero outside the frame
struct alignas(128) SDSlot {
    float sd[2][FH][BW];               // s_i = a_i / den_i and d_i = G.R_i
};
struct alignas(128) GBuf {
    float g[3][FH][BW];                // dL/dRhat
};
struct alignas(128) Slot {
    float4 V[TH][VS];                  // Bt_y(h_i) by field column
};
struct alignas(128) ISlot {
    float I[TH][BBW];                  // I_i at the tile's pixels
};
struct alignas(128) GStage {
    float g[TH][TW];                   // dL/dI_i of the tile, TMA-stored
};
struct Smem {
    GBuf gb[2];
    SDSlot sd[NH];
    Slot slot[NV];
    ISlot is[NB];
    GStage st[2];
    unsigned long long g_full[2], g_empty[2], h_full[NH], h_empty[NH], v_full[NV], v_empty[NV], i_full[NB],
        i_empty[NB];
};

struct BParams {
    const float* rad;    // [N,3,H,W]
    const float* imp;    // [N,M,H,W]
    float* gI;           // [N,M,H,W]
    int N, H, W, M;
    unsigned rpack;      // radius of size i in bits 4i..4i+3
    int debug;           // development switches (env KMD_DEBUG): 1 = no gI stores
};

__device__ __forceinline__ void fuse_bar() { asm volatile("bar.sync 1, %0;" ::"n"(NFUSE * 32) : "memory"); }

__device__ __forceinline__ float4 fma4(float m, float4 a, float4 v) {
    return make_float4(fmaf(m, a.x, v.x), fmaf(m, a.y, v.y), fmaf(m, a.z, v.z), fmaf(m, a.w, v.w));
}

// field: vertical transposed box of h over a column, N = TH outputs, plus the
// folds of the clamped taps at the frame's first / last row (1-D multiplicity
// of source s at q = 0 is R - s + 1, i.e. R - s extra; mirrored at q = H - 1)
template <int R>
__device__ __forceinline__ void field_job(const SDSlot& sd, const GBuf& gb, Slot& sl, int c, int cc, int y0, int H) {
    // h(q) = s(q) (G(q), d(q)) at box row r of this lane's column
    auto hv = [&](int r) {
        const float sv = sd.sd[0][r][cc];
        return make_float4(sv * gb.g[0][r][cc], sv * gb.g[1][r][cc], sv * gb.g[2][r][cc], sv * sd.sd[1][r][cc]);
    };
    float4* Vc = &sl.V[0][c];
    gw_line_field<R, TH>([&](int f) { return hv(RMAX - R + f); }, [&](int oy, float4 v) { Vc[oy * VS] = v; });
    // folds of the clamped taps, only in the frame's first / last tile row (kept
    // out of the Gil-Werman emits: inlining them there bloated the hot code)
    if (y0 == 0) {
        float4 v = Vc[0];
        for (int s = 0; s < R && s < H; ++s) v = fma4((float)(R - s), hv(RMAX + s), v);
        Vc[0] = v;
    }
    if (H - 1 - y0 < TH) {
        const int oy = H - 1 - y0;
        float4 v = Vc[oy * VS];
        for (int s = max(H - R, 0); s < H; ++s) v = fma4((float)(s + R - H + 1), hv(RMAX + s - y0), v);
        Vc[oy * VS] = v;
    }
}

template <int R>
__device__ __forceinline__ void hbox(const Slot& sl, int ty, int xs, float4 (&o)[SEG]) {
    const float4* Vr = &sl.V[ty][xs + RMAX - R];
    gw_line<R, SEG>([&](int j) { return Vr[j]; }, [&](int x, float4 v) { o[x] = v; });
}

__global__ void __launch_bounds__(NTHREADS, 1)
    bwd_t_kernel(const __grid_constant__ BParams p, const __grid_constant__ CUtensorMap tm_sd,
                 const __grid_constant__ CUtensorMap tm_g, const __grid_constant__ CUtensorMap tm_i,
                 const __grid_constant__ CUtensorMap tm_gi, int tiles_x, int tiles_y, int n_tiles) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int M = p.M;
    if (threadIdx.x == 0) {
        for (int b = 0; b < 2; ++b) {
            mbar_init(&sm.g_full[b], 1);
            mbar_init(&sm.g_empty[b], NFIELD);
        }
        for (int s = 0; s < NH; ++s) {
            mbar_init(&sm.h_full[s], 1);
            mbar_init(&sm.h_empty[s], 2);
        }
        for (int s = 0; s < NV; ++s) {
            mbar_init(&sm.v_full[s], 2);
            mbar_init(&sm.v_empty[s], NFUSE);
        }
        for (int s = 0; s < NB; ++s) {
            mbar_init(&sm.i_full[s], 1);
            mbar_init(&sm.i_empty[s], NFUSE);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int my_tiles = n_tiles > (int)blockIdx.x ? (n_tiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    const int per_frame = tiles_x * tiles_y;
    auto tile = [&](int tl, int& n, int& x0, int& y0) {
        const int t = blockIdx.x + tl * gridDim.x;
        n = t / per_frame;
        const int r = t - n * per_frame, ty = r / tiles_x;
        x0 = (r - ty * tiles_x) * TW;
        y0 = ty * TH;
    };

    if (warp == 0) {
        if (lane == 0) {
            for (int tl = 0; tl < my_tiles; ++tl) {
                int n, x0, y0;
                tile(tl, n, x0, y0);
                const int gbi = tl & 1;
                mbar_wait(&sm.g_empty[gbi], ((tl >> 1) & 1) ^ 1);
                mbar_arrive_expect_tx(&sm.g_full[gbi], 3 * FH * BW * 4);
                tma_load_3d(&sm.gb[gbi].g[0][0][0], &tm_g, x0 - XOFF, y0 - RMAX, 3 * n, &sm.g_full[gbi]);
                for (int i = 0; i < M; ++i) {
                    const int seq = tl * M + i, sh = seq % NH, sb = seq % NB;
                    mbar_wait(&sm.h_empty[sh], ((seq / NH) & 1) ^ 1);
                    mbar_arrive_expect_tx(&sm.h_full[sh], 2 * FH * BW * 4);
                    tma_load_3d(&sm.sd[sh].sd[0][0][0], &tm_sd, x0 - XOFF, y0 - RMAX, 2 * (n * M + i), &sm.h_full[sh]);
                    mbar_wait(&sm.i_empty[sb], ((seq / NB) & 1) ^ 1);
                    mbar_arrive_expect_tx(&sm.i_full[sb], TH * BBW * 4);
                    tma_load_3d(&sm.is[sb].I[0][0], &tm_i, x0, y0, n * M + i, &sm.i_full[sb]);
                }
            }
        }
    } else if (warp <= NFIELD) {
        const int fw = warp - 1;
        for (int tl = 0; tl < my_tiles; ++tl) {
            int n, x0, y0;
            tile(tl, n, x0, y0);
            (void)n;
            const int gbi = tl & 1;
            mbar_wait(&sm.g_full[gbi], (tl >> 1) & 1);
#pragma unroll 1
            for (int jl = fw; jl < 2 * M; jl += NFIELD) {
                const int i = jl >> 1, h = jl & 1;
                const int seq = tl * M + i, sh = seq % NH, sv = seq % NV;
                // field column c <-> global x0 - 6 + c <-> box column c + 2
                // (unclamped: zero outside the frame)
                const int c = h * 32 + lane, cc = c + XOFF - RMAX;
                mbar_wait(&sm.v_empty[sv], ((seq / NV) & 1) ^ 1);
                mbar_wait(&sm.h_full[sh], (seq / NH) & 1);
                const SDSlot& sd = sm.sd[sh];
                const GBuf& gb = sm.gb[gbi];
                switch ((p.rpack >> (4 * i)) & 15) {
                    case 0: field_job<0>(sd, gb, sm.slot[sv], c, cc, y0, p.H); break;
                    case 1: field_job<1>(sd, gb, sm.slot[sv], c, cc, y0, p.H); break;
                    case 2: field_job<2>(sd, gb, sm.slot[sv], c, cc, y0, p.H); break;
                    case 3: field_job<3>(sd, gb, sm.slot[sv], c, cc, y0, p.H); break;
                    case 4: field_job<4>(sd, gb, sm.slot[sv], c, cc, y0, p.H); break;
                    case 5: field_job<5>(sd, gb, sm.slot[sv], c, cc, y0, p.H); break;
                    default: field_job<6>(sd, gb, sm.slot[sv], c, cc, y0, p.H); break;
                }
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(&sm.h_empty[sh]);
                    mbar_arrive(&sm.v_full[sv]);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.g_empty[gbi]);
        }
    } else {
        const int c = threadIdx.x - (1 + NFIELD) * 32;
        const int ty = c / NSEG, sub = c % NSEG;
        const bool active = ty < TH;
        const int xs = (0x2d27211a130c0600ull >> (8 * sub)) & 0xff;
        const int len = (0x76677766u >> (4 * sub)) & 0xf;
        const size_t plane = (size_t)p.H * p.W;
        int vs = 0, vph = 0, bs = 0, bph = 0, sb2 = 0;
        for (int tl = 0; tl < my_tiles; ++tl) {
            int n, x0, y0;
            tile(tl, n, x0, y0);
            const int gy = y0 + ty, gyc = min(gy, p.H - 1);
            const bool row_ok = active && gy < p.H;
            const bool edge_x = x0 == 0 || x0 + TW >= p.W;
            float rr[SEG][3];
            const float* rp = p.rad + (size_t)n * 3 * plane + (size_t)gyc * p.W;
#pragma unroll
            for (int j = 0; j < SEG; ++j) {
                const int gx = min(x0 + xs + j, p.W - 1);
                rr[j][0] = __ldg(rp + gx);
                rr[j][1] = __ldg(rp + plane + gx);
                rr[j][2] = __ldg(rp + 2 * plane + gx);
            }
#pragma unroll 1
            for (int i = 0; i < M; ++i) {
                mbar_wait(&sm.v_full[vs], vph);
                mbar_wait(&sm.i_full[bs], bph);
                if (active) {
                    const int R = (p.rpack >> (4 * i)) & 15;
                    const Slot& sl = sm.slot[vs];
                    float4 o[SEG];
                    switch (R) {
                        case 0: hbox<0>(sl, ty, xs, o); break;
                        case 1: hbox<1>(sl, ty, xs, o); break;
                        case 2: hbox<2>(sl, ty, xs, o); break;
                        case 3: hbox<3>(sl, ty, xs, o); break;
                        case 4: hbox<4>(sl, ty, xs, o); break;
                        case 5: hbox<5>(sl, ty, xs, o); break;
                        default: hbox<6>(sl, ty, xs, o); break;
                    }
                    const float* Ir = &sm.is[bs].I[ty][xs];
                    float* go = &sm.st[sb2].g[ty][xs];
#pragma unroll
                    for (int j = 0; j < SEG; ++j) {
                        const int gx = x0 + xs + j;
                        if (j < len) {
                            float4 v = o[j];
                            if (edge_x && row_ok) {  // horizontal folds at the frame's first / last column
                                if (gx == 0)
                                    for (int s = 0; s < R && s < p.W; ++s)
                                        v = fma4((float)(R - s), sl.V[ty][s - x0 + RMAX], v);
                                if (gx == p.W - 1)
                                    for (int s = max(p.W - R, 0); s < p.W; ++s)
                                        v = fma4((float)(s + R - p.W + 1), sl.V[ty][s - x0 + RMAX], v);
                            }
                            const float e = exp_acc(Ir[j]);
                            go[j] = e * (fmaf(rr[j][0], v.x, fmaf(rr[j][1], v.y, rr[j][2] * v.z)) - v.w);
                        }
                    }
                }
                __syncwarp();
                if ((c & 31) == 0) {
                    mbar_arrive(&sm.v_empty[vs]);
                    mbar_arrive(&sm.i_empty[bs]);
                }
                // the tile's dL/dI_i leaves with one TMA store (clipped at the frame
                // edge); double-buffered stage: before the barrier, the store of
                // the previous step must have read its buffer (reused next step)
                fence_proxy_async();
                if (c == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                fuse_bar();
                if (c == 0 && !(p.debug & 1)) tma_store_3d(&tm_gi, x0, y0, n * M + i, &sm.st[sb2].g[0][0]);
                sb2 ^= 1;
                if (++vs == NV) { vs = 0; vph ^= 1; }
                if (++bs == NB) { bs = 0; bph ^= 1; }
            }
        }
        if (c == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

// Log-sum-exp of the M logits per pixel, L = m + log sum_i exp(B_i - m),
// m = max_i B_i, for pass A's softmax weights a_i = exp(B_i - L) (Eq. 5,
// PAPER.md:251).  Four pixels per thread (plane % 4 == 0 on the TMA path).
__global__ void __launch_bounds__(256) lse_kernel(const float* __restrict__ blend, float* __restrict__ lse, int M,
                                                  int plane) {
    const int nq = plane / 4;
    const size_t f0 = (size_t)blockIdx.y * M * plane;
    for (int t = blockIdx.x * 256 + threadIdx.x; t < nq; t += gridDim.x * 256) {
        float4 b[KMD_MAX_SIZES];
#pragma unroll
        for (int i = 0; i < KMD_MAX_SIZES; ++i) {
            if (i >= M) break;
            b[i] = __ldg(reinterpret_cast<const float4*>(blend + f0 + (size_t)i * plane) + t);
        }
        float4 m = b[0];
#pragma unroll
        for (int i = 1; i < KMD_MAX_SIZES; ++i) {
            if (i >= M) break;
            m = make_float4(fmaxf(m.x, b[i].x), fmaxf(m.y, b[i].y), fmaxf(m.z, b[i].z), fmaxf(m.w, b[i].w));
        }
        float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int i = 0; i < KMD_MAX_SIZES; ++i) {
            if (i >= M) break;
            s.x += expf(b[i].x - m.x);
            s.y += expf(b[i].y - m.y);
            s.z += expf(b[i].z - m.z);
            s.w += expf(b[i].w - m.w);
        }
        reinterpret_cast<float4*>(lse + (size_t)blockIdx.y * plane)[t] =
            make_float4(m.x + logf(s.x), m.y + logf(s.y), m.z + logf(s.z), m.w + logf(s.w));
    }
}

// pass C: dL/dB_i = a_i (G.R_i - sum_j a_j G.R_j), a = softmax(B) (logits).
// One thread per 4 consecutive pixels of a frame (float4 when plane % 4 == 0);
// blockIdx.y = frame, so no 64-bit division per element.
template <bool VEC>
__global__ void __launch_bounds__(256) bwd_blend_kernel(const float* __restrict__ blend, const float* __restrict__ ws,
                                                        float* __restrict__ gB, int M, int plane) {
    const int nq = (plane + 3) / 4;
    const size_t f0 = (size_t)blockIdx.y * M * plane;
    for (int t = blockIdx.x * 256 + threadIdx.x; t < nq; t += gridDim.x * 256) {
        const int q0 = 4 * t, cnt = min(4, plane - q0);
        float bv[KMD_MAX_SIZES][4], d[KMD_MAX_SIZES][4];
#pragma unroll
        for (int i = 0; i < KMD_MAX_SIZES; ++i) {
            if (i >= M) break;
            const float* bp = blend + f0 + (size_t)i * plane + q0;
            const float* gp = ws + 2 * (f0 + (size_t)i * plane) + plane + q0;  // d_i of [N*M][2][H][W]
            if (VEC) {
                const float4 x = __ldg(reinterpret_cast<const float4*>(bp));
                const float4 y = __ldg(reinterpret_cast<const float4*>(gp));
                bv[i][0] = x.x, bv[i][1] = x.y, bv[i][2] = x.z, bv[i][3] = x.w;
                d[i][0] = y.x, d[i][1] = y.y, d[i][2] = y.z, d[i][3] = y.w;
            } else {
                for (int k = 0; k < 4; ++k) {
                    bv[i][k] = k < cnt ? __ldg(bp + k) : 0.f;
                    d[i][k] = k < cnt ? __ldg(gp + k) : 0.f;
                }
            }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            float m = -INFINITY;
#pragma unroll
            for (int i = 0; i < KMD_MAX_SIZES; ++i)
                if (i < M) m = fmaxf(m, bv[i][k]);
            float sum = 0.f, mean = 0.f;
#pragma unroll
            for (int i = 0; i < KMD_MAX_SIZES; ++i)
                if (i < M) {
                    bv[i][k] = expf(bv[i][k] - m);
                    sum += bv[i][k];
                    mean = fmaf(bv[i][k], d[i][k], mean);
                }
            const float inv = 1.f / sum;
            mean *= inv;
#pragma unroll
            for (int i = 0; i < KMD_MAX_SIZES; ++i)
                if (i < M) d[i][k] = bv[i][k] * inv * (d[i][k] - mean);
        }
#pragma unroll
        for (int i = 0; i < KMD_MAX_SIZES; ++i) {
            if (i >= M) break;
            float* gp = gB + f0 + (size_t)i * plane + q0;
            if (VEC) {
                *reinterpret_cast<float4*>(gp) = make_float4(d[i][0], d[i][1], d[i][2], d[i][3]);
            } else {
                for (int k = 0; k < cnt; ++k) gp[k] = d[i][k];
            }
        }
    }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn get_encode() {
    static EncodeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(f);
    });
    return fn;
}

bool encode(CUtensorMap* m, int rank, const void* base, const cuuint64_t* dims, const cuuint64_t* strides,
            const cuuint32_t* box) {
    EncodeFn enc = get_encode();
    if (!enc) return false;
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, const_cast<void*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace bwd

bool bwd_tma_supported(int H, int W, int M, const int* sizes, const void* a, const void* b, const void* c,
                       const void* d) {
    if (M < 1 || M > KMD_MAX_SIZES || W % 4 != 0) return false;
    for (int i = 0; i < M; ++i)
        if ((sizes[i] - 1) / 2 > bwd::RMAX) return false;
    if (((uintptr_t)a | (uintptr_t)b | (uintptr_t)c | (uintptr_t)d) & 15) return false;
    (void)H;
    return bwd::get_encode() != nullptr;
}

// (s_i, d_i) per pixel and size: [N*M][2][H][W] floats
// (s_i, d_i) planes [N*M][2][H][W], then the log-sum-exp plane [N][H][W]
size_t bwd_tma_workspace_bytes(int N, int H, int W, int M) {
    return ((size_t)N * M * H * W * 2 + (size_t)N * H * W) * sizeof(float);
}

cudaError_t launch_backward_tma(const float* rad, const float* imp, const float* blend, const float* G, float* gI,
                                float* gB, int N, int H, int W, int M, const int* sizes, int logits, void* ws,
                                cudaStream_t st) {
    using namespace bwd;
    float* sd = reinterpret_cast<float*>(ws);
    // ---- pass A: (s_i, d_i) (the forward kernel's tiles and box sums)
    FusedParams p{};
    p.rad = rad;
    p.imp = imp;
    p.blend = M > 1 ? blend : nullptr;
    p.N = N;
    p.W = W;
    p.H = H;
    p.row_base = 0;
    p.buf_rows = H;
    p.out_y0 = 0;
    p.out_rows = H;
    p.M = M;
    p.blend_is_logits = logits;
    unsigned rpack = 0;
    int rmax = 0;
    for (int i = 0; i < KMD_MAX_SIZES; ++i) p.sizes[i] = i < M ? sizes[i] : 1;
    for (int i = 0; i < M; ++i) {
        const int r = (sizes[i] - 1) / 2;
        rmax = r > rmax ? r : rmax;
        rpack |= (unsigned)r << (4 * i);
    }
    p.rmax = rmax;
    p.grad = G;
    if (M > 1 && logits) {
        // ---- log-sum-exp of the logits per pixel (pass A's softmax weights)
        float* lse = sd + (size_t)N * M * H * W * 2;
        const int plane = H * W, nq = plane / 4;
        int dev0 = 0, sms0 = 148;
        cudaGetDevice(&dev0);
        cudaDeviceGetAttribute(&sms0, cudaDevAttrMultiProcessorCount, dev0);
        const int gx = (nq + 255) / 256 < sms0 * 8 ? (nq + 255) / 256 : sms0 * 8;
        lse_kernel<<<dim3(gx, N), 256, 0, st>>>(blend, lse, M, plane);
        cudaError_t e0 = cudaGetLastError();
        if (e0 != cudaSuccess) return e0;
        p.lse = lse;
    }
    static const int dbg = [] { const char* s = getenv("KMD_DEBUG"); return s ? atoi(s) : 0; }();
    p.debug = dbg;
    cudaError_t e = launch_bwd_h_tma(p, sd, st);
    if (e != cudaSuccess) return e;
    // ---- pass B: transposed box of h_i = s_i (G, d_i), dL/dI_i
    BParams q{rad, imp, gI, N, H, W, M, rpack, dbg};
    CUtensorMap m_sd, m_g, m_i;
    {
        const cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, 2 * (cuuint64_t)N * M};
        const cuuint64_t strides[2] = {(cuuint64_t)W * 4, (cuuint64_t)W * H * 4};
        const cuuint32_t box[3] = {BW, FH, 2};
        if (!encode(&m_sd, 3, sd, dims, strides, box)) return cudaErrorInvalidValue;
    }
    {
        const cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, 3 * (cuuint64_t)N};
        const cuuint64_t strides[2] = {(cuuint64_t)W * 4, (cuuint64_t)W * H * 4};
        const cuuint32_t box[3] = {BW, FH, 3};
        if (!encode(&m_g, 3, G, dims, strides, box)) return cudaErrorInvalidValue;
    }
    CUtensorMap m_gi;
    {
        const cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N * M};
        const cuuint64_t strides[2] = {(cuuint64_t)W * 4, (cuuint64_t)W * H * 4};
        const cuuint32_t box[3] = {BBW, TH, 1};
        if (!encode(&m_i, 3, imp, dims, strides, box)) return cudaErrorInvalidValue;
        const cuuint32_t obox[3] = {TW, TH, 1};
        if (!encode(&m_gi, 3, gI, dims, strides, obox)) return cudaErrorInvalidValue;
    }
    const int tiles_y = (H + TH - 1) / TH, tiles_x = (W + TW - 1) / TW;
    const long long n_tiles = (long long)tiles_x * tiles_y * N;
    if (n_tiles > 0x7fffffff) return cudaErrorInvalidValue;
    int dev = 0, sms = 148;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
    if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
    const size_t smem = sizeof(Smem);
    if ((e = cudaFuncSetAttribute(bwd_t_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) !=
        cudaSuccess)
        return e;
    const int grid = (int)(n_tiles < sms ? n_tiles : sms);
    bwd_t_kernel<<<grid, NTHREADS, smem, st>>>(q, m_sd, m_g, m_i, m_gi, tiles_x, tiles_y, (int)n_tiles);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    // ---- pass C: dL/dB
    if (gB && M == 1) return cudaMemsetAsync(gB, 0, sizeof(float) * (size_t)N * H * W, st);
    if (gB && logits) {
        const int plane = H * W, nq = (plane + 3) / 4;
        const int gx = (nq + 255) / 256 < sms * 8 ? (nq + 255) / 256 : sms * 8;
        const dim3 grid(gx, N);
        const bool vec = plane % 4 == 0 && (((uintptr_t)blend | (uintptr_t)gB) & 15) == 0;
        if (vec) bwd_blend_kernel<true><<<grid, 256, 0, st>>>(blend, sd, gB, M, plane);
        else bwd_blend_kernel<false><<<grid, 256, 0, st>>>(blend, sd, gB, M, plane);
        return cudaGetLastError();
    }
    if (gB)  // alpha given: dL/dalpha_i = G.R_i = d_i, every second plane of the workspace
        return cudaMemcpy2DAsync(gB, (size_t)H * W * 4, sd + (size_t)H * W, 2 * (size_t)H * W * 4,
                                 (size_t)H * W * 4, (size_t)N * M, cudaMemcpyDeviceToDevice, st);
    return cudaSuccess;
}

}  // namespace kmd
