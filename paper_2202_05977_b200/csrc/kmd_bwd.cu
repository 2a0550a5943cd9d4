// kmd_bwd.cu -- NEXT row 3: gradients of the reconstruction w.r.t. the
// importance maps and the fusion logits (end-to-end training through the
// decoder, Eq. 1, 614).
//
// With G = dL/dRhat, alpha = softmax(B), e_i = exp(I_i), den_i / num_i the k_i
// box sums of e_i and e_i r (the forward's ratio-of-box form):
//   dL/dB_i(p)  = alpha_i(p) sum_c G_c(p) (R_i,c(p) - Rhat_c(p))          (softmax Jacobian)
//   g_i,c(p)    = alpha_i(p) G_c(p)                                      (dL/dR_i)
//   dL/dI_i(q)  = e_i(q) [ sum_c r_c(q) Bt(g_i,c / den_i)(q) - Bt(sum_c g_i,c R_i,c / den_i)(q) ]
// where Bt is the transpose of the clamp-to-edge k x k box: a plain box sum in
// the interior (with the field zero outside the frame), plus the clamped taps
// folded back onto the border pixels (1-D multiplicity of source p at q = 0 is
// r - p + 1, mirrored at q = n - 1).  Separable: Bt = Bt_x o Bt_y.
//
// One 512-thread CTA per 32 x 64 output tile and frame (16 warps: every pass is
// bound by shared-memory and L2 latency, so occupancy is what pays); per size
// i (radius r):
//   1. P = (e, e r, e g, e b) over the tile + 2r halo (clamped source pixels),
//      elementwise into shared memory;
//   2. vertical box sums of P (Gil-Werman, one thread per column);
//   3. horizontal box sums -> S = (den, num) over the tile + r halo; there
//      h = (alpha G / den, alpha G.R / den) (0 outside the frame), and
//      G.R_i at the tile's pixels is parked in grad_blend;
//   4. Bt vertical (Gil-Werman over h, plus the border folds);
//   5. Bt horizontal, then dL/dI_i = e (r . T - T_R) at the tile's pixels.
// After the last size, dL/dB_i = alpha_i (G.R_i - sum_j alpha_j G.R_j).
// Unshifted exp: importance must lie in (-80, 80) (header note).
#include "kmd_gw.cuh"
#include "kmd_kernels.h"

namespace kmd {
namespace {

constexpr int RMAX = 6;
constexpr int TQH = 32, TQW = 64;                 // output tile
constexpr int SH = TQH + 2 * RMAX;                // 44: rows of the S / h region
constexpr int PH = TQH + 4 * RMAX;                // 56: rows of the P region
constexpr int PS = 96;                            // row stride of P / V / h buffers (>= 64 + 4 RMAX + 8)
constexpr int SEGB = 4;                           // outputs per thread in every box pass
constexpr int NT = 512;                           // 16 warps: the passes are latency-bound

struct BwdSmem {
    float4 V[SH][PS];                             // vertical box sums of P; later Bt_y(h)
    union {
        float4 P[PH][PS];                         // premultiplied field
        float4 h[SH][PS];                         // per-pixel gradient field
    } u;
    float mB[SH][TQW + 2 * RMAX];                 // softmax shift and 1 / sum over the S region
    float iB[SH][TQW + 2 * RMAX];
};

struct BwdParams {
    const float *rad, *imp, *blend, *G;
    float *gI, *gB;
    int H, W, M, logits;
    unsigned rpack;                               // radius of size i in bits 4i..4i+3
};

template <int R>
__device__ __forceinline__ void size_pass(const BwdParams& p, BwdSmem& sm, int n, int i, int y0, int x0) {
    const int tid = threadIdx.x;
    const size_t plane = (size_t)p.H * p.W;
    const float* rad = p.rad + (size_t)n * 3 * plane;
    const float* Ii = p.imp + ((size_t)n * p.M + i) * plane;
    const float* Gn = p.G + (size_t)n * 3 * plane;
    constexpr int PW = TQW + 4 * R, PR = TQH + 4 * R;   // P region (rows y0-2R.., cols x0-2R..)
    constexpr int SWd = TQW + 2 * R, SR = TQH + 2 * R;  // S region (rows y0-R.., cols x0-R..)

    // 1. P over the P region, clamp-to-edge sources (reading R1); unrolled so
    // that several elements' global loads are in flight at once
#pragma unroll 4
    for (int e = tid; e < PR * PW; e += NT) {
        const int rr = e / PW, cc = e - rr * PW;
        const int gy = clampi(y0 - 2 * R + rr, 0, p.H - 1), gx = clampi(x0 - 2 * R + cc, 0, p.W - 1);
        const size_t q = (size_t)gy * p.W + gx;
        const float ev = expf(__ldg(Ii + q));
        sm.u.P[rr][cc] = make_float4(ev, ev * __ldg(rad + q), ev * __ldg(rad + plane + q), ev * __ldg(rad + 2 * plane + q));
    }
    __syncthreads();
    // 2. vertical sums: V[j][c] = sum_{f=j}^{j+2R} P[f][c], j < SR
    // (column, 8-row segment) items keep every thread busy; the reads past the
    // last P row of the final segment stay inside the shared block and feed
    // only outputs that are not stored
    constexpr int VSEGS = (SR + SEGB - 1) / SEGB;
    for (int it = tid; it < PW * VSEGS; it += NT) {
        const int c = it % PW, j0 = (it / PW) * SEGB;
        gw_line<R, SEGB>([&](int f) { return sm.u.P[j0 + f][c]; }, [&](int t, float4 v) {
            if (j0 + t < SR) sm.V[j0 + t][c] = v;
        });
    }
    __syncthreads();
    // 3. horizontal sums -> S; h and G.R_i
    constexpr int NSEGS = (SWd + SEGB - 1) / SEGB;
    for (int it = tid; it < SR * NSEGS; it += NT) {
        const int j = it / NSEGS, k0 = (it - j * NSEGS) * SEGB;
        const int gy = y0 - R + j;
        const bool row_in = gy >= 0 && gy < p.H;
        // issue this segment's global loads (G, logit) before the box sums so
        // their latency overlaps the shared-memory work
        float gl[SEGB][3], bl[SEGB];
        const float* Bi = p.M > 1 ? p.blend + ((size_t)n * p.M + i) * plane : nullptr;
#pragma unroll
        for (int t = 0; t < SEGB; ++t) {
            const int gx = x0 - R + k0 + t;
            const bool in = row_in && gx >= 0 && gx < p.W && k0 + t < SWd;
            const size_t q = in ? (size_t)gy * p.W + gx : 0;
            gl[t][0] = in ? __ldg(Gn + q) : 0.f;
            gl[t][1] = in ? __ldg(Gn + plane + q) : 0.f;
            gl[t][2] = in ? __ldg(Gn + 2 * plane + q) : 0.f;
            bl[t] = (in && Bi) ? __ldg(Bi + q) : 0.f;
        }
        float4 S[SEGB];
        gw_line<R, SEGB>([&](int t) { return sm.V[j][k0 + t]; }, [&](int t, float4 v) { S[t] = v; });
#pragma unroll
        for (int t = 0; t < SEGB; ++t) {
            const int k = k0 + t;
            if (k >= SWd) break;
            const int gx = x0 - R + k;
            float4 hval = make_float4(0.f, 0.f, 0.f, 0.f);
            if (row_in && gx >= 0 && gx < p.W) {
                const size_t q = (size_t)gy * p.W + gx;
                const float rden = 1.f / S[t].x;
                const float R0 = S[t].y * rden, R1 = S[t].z * rden, R2 = S[t].w * rden;
                float a = 1.f;
                if (p.M > 1)
                    a = p.logits ? expf(bl[t] - sm.mB[j + RMAX - R][k + RMAX - R]) * sm.iB[j + RMAX - R][k + RMAX - R]
                                 : bl[t];
                const float g0 = gl[t][0], g1 = gl[t][1], g2 = gl[t][2];
                const float ar = a * rden;
                const float dot = g0 * R0 + g1 * R1 + g2 * R2;
                hval = make_float4(ar * g0, ar * g1, ar * g2, ar * dot);
                const int ty = j - R, tx = k - R;
                if (p.gB && ty >= 0 && ty < TQH && tx >= 0 && tx < TQW)
                    p.gB[((size_t)n * p.M + i) * plane + q] = dot;  // G.R_i, finished below
            }
            sm.u.h[j][k] = hval;
        }
    }
    __syncthreads();
    // 4. Bt vertical: V[t][k] = sum_{j=t}^{t+2R} h[j][k] (+ folds at the frame's top / bottom row)
    for (int it = tid; it < SWd * (TQH / SEGB); it += NT) {
        const int k = it % SWd, t0 = (it / SWd) * SEGB;
        gw_line<R, SEGB>([&](int f) { return sm.u.h[t0 + f][k]; }, [&](int tt, float4 v) {
            const int t = t0 + tt;
            const int gy = y0 + t;
            // (H == 1 takes both folds: 1 + R + R = 2R + 1 taps on the one row)
            if (gy == 0) {
                // sources p = 0 .. R-1 (h rows j = p + R - y0) land R - p extra times
                for (int s = 0; s < R; ++s) {
                    const float4 hs = sm.u.h[s + R][k];
                    const float m = (float)(R - s);
                    v = make_float4(fmaf(m, hs.x, v.x), fmaf(m, hs.y, v.y), fmaf(m, hs.z, v.z), fmaf(m, hs.w, v.w));
                }
            }
            if (gy == p.H - 1) {
                for (int s = p.H - R; s < p.H; ++s) {
                    if (s < 0) continue;
                    const float4 hs = sm.u.h[s - y0 + R][k];
                    const float m = (float)(s + R - p.H + 1);
                    v = make_float4(fmaf(m, hs.x, v.x), fmaf(m, hs.y, v.y), fmaf(m, hs.z, v.z), fmaf(m, hs.w, v.w));
                }
            }
            sm.V[t][k] = v;
        });
    }
    __syncthreads();
    // 5. Bt horizontal and dL/dI_i at the tile's pixels
    constexpr int QSEGS = TQW / SEGB;
#pragma unroll 2
    for (int it = tid; it < TQH * QSEGS; it += NT) {
        const int t = it / QSEGS, u0 = (it - t * QSEGS) * SEGB;
        float4 T[SEGB];
        gw_line<R, SEGB>([&](int f) { return sm.V[t][u0 + f]; }, [&](int f, float4 v) { T[f] = v; });
        const int gy = y0 + t;
        if (gy >= p.H) continue;
#pragma unroll
        for (int f = 0; f < SEGB; ++f) {
            const int gx = x0 + u0 + f;
            if (gx >= p.W) break;
            float4 v = T[f];
            if (gx == 0) {
                for (int s = 0; s < R; ++s) {
                    const float4 hs = sm.V[t][s + R - x0];
                    const float m = (float)(R - s);
                    v = make_float4(fmaf(m, hs.x, v.x), fmaf(m, hs.y, v.y), fmaf(m, hs.z, v.z), fmaf(m, hs.w, v.w));
                }
            }
            if (gx == p.W - 1) {
                for (int s = p.W - R; s < p.W; ++s) {
                    if (s < 0) continue;
                    const float4 hs = sm.V[t][s - x0 + R];
                    const float m = (float)(s + R - p.W + 1);
                    v = make_float4(fmaf(m, hs.x, v.x), fmaf(m, hs.y, v.y), fmaf(m, hs.z, v.z), fmaf(m, hs.w, v.w));
                }
            }
            const size_t q = (size_t)gy * p.W + gx;
            const float ev = expf(__ldg(Ii + q));
            const float s = __ldg(rad + q) * v.x + __ldg(rad + plane + q) * v.y + __ldg(rad + 2 * plane + q) * v.z - v.w;
            p.gI[((size_t)n * p.M + i) * plane + q] = ev * s;
        }
    }
    __syncthreads();
}

__global__ void __launch_bounds__(NT, 1) bwd_tile_kernel(const BwdParams p, int tiles_x, int tiles_y) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    BwdSmem& sm = *reinterpret_cast<BwdSmem*>(smem_raw);
    const int per = tiles_x * tiles_y;
    const int n = blockIdx.x / per, r = blockIdx.x - n * per;
    const int y0 = (r / tiles_x) * TQH, x0 = (r % tiles_x) * TQW;
    const size_t plane = (size_t)p.H * p.W;
    // softmax shift and normaliser of the logits over the S region (R = RMAX)
    if (p.M > 1 && p.logits) {
        for (int e = threadIdx.x; e < SH * (TQW + 2 * RMAX); e += NT) {
            const int j = e / (TQW + 2 * RMAX), k = e - j * (TQW + 2 * RMAX);
            const int gy = y0 - RMAX + j, gx = x0 - RMAX + k;
            float m = 0.f, s = 1.f;
            if (gy >= 0 && gy < p.H && gx >= 0 && gx < p.W) {
                const float* b = p.blend + (size_t)n * p.M * plane + (size_t)gy * p.W + gx;
                float bv[KMD_MAX_SIZES];
#pragma unroll
                for (int i = 0; i < KMD_MAX_SIZES; ++i) bv[i] = i < p.M ? __ldg(b + i * plane) : -INFINITY;
                m = -INFINITY;
#pragma unroll
                for (int i = 0; i < KMD_MAX_SIZES; ++i) m = fmaxf(m, bv[i]);
                s = 0.f;
#pragma unroll
                for (int i = 0; i < KMD_MAX_SIZES; ++i) s += i < p.M ? expf(bv[i] - m) : 0.f;
            }
            sm.mB[j][k] = m;
            sm.iB[j][k] = 1.f / s;
        }
    }
    __syncthreads();
    for (int i = 0; i < p.M; ++i) {
        switch ((p.rpack >> (4 * i)) & 15) {
            case 0: size_pass<0>(p, sm, n, i, y0, x0); break;
            case 1: size_pass<1>(p, sm, n, i, y0, x0); break;
            case 2: size_pass<2>(p, sm, n, i, y0, x0); break;
            case 3: size_pass<3>(p, sm, n, i, y0, x0); break;
            case 4: size_pass<4>(p, sm, n, i, y0, x0); break;
            case 5: size_pass<5>(p, sm, n, i, y0, x0); break;
            default: size_pass<6>(p, sm, n, i, y0, x0); break;
        }
    }
    // dL/dB_i = alpha_i (G.R_i - sum_j alpha_j G.R_j)   (logits); G.R_i as is (alpha given)
    if (p.gB && p.M > 1 && p.logits) {
        for (int e = threadIdx.x; e < TQH * TQW; e += NT) {
            const int t = e / TQW, u = e - t * TQW, gy = y0 + t, gx = x0 + u;
            if (gy >= p.H || gx >= p.W) continue;
            const size_t q = (size_t)gy * p.W + gx;
            const float* b = p.blend + (size_t)n * p.M * plane + q;
            float* gb = p.gB + (size_t)n * p.M * plane + q;
            const float m = sm.mB[t + RMAX][u + RMAX], is = sm.iB[t + RMAX][u + RMAX];
            float a[KMD_MAX_SIZES], d[KMD_MAX_SIZES];
#pragma unroll
            for (int i = 0; i < KMD_MAX_SIZES; ++i) {
                a[i] = i < p.M ? __ldg(b + i * plane) : 0.f;
                d[i] = i < p.M ? gb[i * plane] : 0.f;
            }
            float mean = 0.f;
#pragma unroll
            for (int i = 0; i < KMD_MAX_SIZES; ++i) {
                a[i] = i < p.M ? expf(a[i] - m) * is : 0.f;
                mean = fmaf(a[i], d[i], mean);
            }
#pragma unroll
            for (int i = 0; i < KMD_MAX_SIZES; ++i)
                if (i < p.M) gb[i * plane] = a[i] * (d[i] - mean);
        }
    }
}

}  // namespace

size_t bwd_workspace_floats(int, int, int) { return 0; }

cudaError_t launch_backward(const float* rad, const float* imp, const float* blend, const float* G, float* gI,
                            float* gB, int N, int H, int W, int M, const int* sizes, int logits, float*,
                            cudaStream_t st) {
    BwdParams p;
    p.rad = rad;
    p.imp = imp;
    p.blend = blend;
    p.G = G;
    p.gI = gI;
    p.gB = gB;
    p.H = H;
    p.W = W;
    p.M = M;
    p.logits = logits;
    p.rpack = 0;
    for (int i = 0; i < M; ++i) {
        const int r = (sizes[i] - 1) / 2;
        if (r > RMAX) return cudaErrorInvalidValue;
        p.rpack |= (unsigned)r << (4 * i);
    }
    if (gB && M == 1) {
        cudaError_t e = cudaMemsetAsync(gB, 0, sizeof(float) * (size_t)N * H * W, st);
        if (e != cudaSuccess) return e;
        p.gB = nullptr;
    }
    const int tiles_x = (W + TQW - 1) / TQW, tiles_y = (H + TQH - 1) / TQH;
    const long long blocks = (long long)tiles_x * tiles_y * N;
    if (blocks > 0x7fffffff) return cudaErrorInvalidValue;
    const size_t smem = sizeof(BwdSmem);
    cudaError_t e = cudaFuncSetAttribute(bwd_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    bwd_tile_kernel<<<(int)blocks, NT, smem, st>>>(p, tiles_x, tiles_y);
    return cudaGetLastError();
}

}  // namespace kmd
