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
// the interior, with the clamped taps folded back onto the border pixels
// (1-D multiplicity of source p at border q: r - p + 1 at q = 0, mirrored at
// q = n - 1).  Separable: Bt = Bt_x o Bt_y.
//
// Straightforward kernels (one thread per pixel, shared nothing); the
// backward is not on the timed hot path.
#include "kmd_kernels.h"

namespace kmd {
namespace {

constexpr int NT = 256;

int blocks_for(long long n) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    long long b = (n + NT - 1) / NT;
    const long long cap = (long long)sms * 16;
    return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

// forward box sums of size k for one map: S(p) = sum_{q in Omega_k(p)} (e, e r, e g, e b)(q),
// clamp-to-edge.  Pass 1 (axis 0 = vertical) builds the premultiplied field on the fly.
__global__ void __launch_bounds__(NT) box_fwd_v(const float* __restrict__ rad, const float* __restrict__ imp,
                                                float4* __restrict__ out, int H, int W, int r) {
    const long long total = (long long)H * W;
    for (long long t = blockIdx.x * (long long)NT + threadIdx.x; t < total; t += (long long)gridDim.x * NT) {
        const int y = (int)(t / W), x = (int)(t - (long long)y * W);
        float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int dy = -r; dy <= r; ++dy) {
            const long long q = (long long)min(max(y + dy, 0), H - 1) * W + x;
            const float e = expf(__ldg(imp + q));
            s.x += e;
            s.y = fmaf(e, __ldg(rad + q), s.y);
            s.z = fmaf(e, __ldg(rad + total + q), s.z);
            s.w = fmaf(e, __ldg(rad + 2 * total + q), s.w);
        }
        out[t] = s;
    }
}

__global__ void __launch_bounds__(NT) box_h(const float4* __restrict__ in, float4* __restrict__ out, int H, int W,
                                            int r) {
    const long long total = (long long)H * W;
    for (long long t = blockIdx.x * (long long)NT + threadIdx.x; t < total; t += (long long)gridDim.x * NT) {
        const int y = (int)(t / W), x = (int)(t - (long long)y * W);
        float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int dx = -r; dx <= r; ++dx) {
            const float4 v = in[(long long)y * W + min(max(x + dx, 0), W - 1)];
            s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
        }
        out[t] = s;
    }
}

// per-pixel part: softmax of the logits, Rhat, dL/dB, and the two fields to be
// transposed-box-filtered for dL/dI (stored per size as float4 (h_r, h_g, h_b, h_R)).
__global__ void __launch_bounds__(NT) pixel_bwd(const float4* __restrict__ S /*[M][HW]*/,
                                                const float* __restrict__ blend /*[M][HW] or null*/,
                                                const float* __restrict__ G /*[3][HW]*/, float* __restrict__ gB,
                                                float4* __restrict__ h /*[M][HW]*/, int M, long long HW,
                                                int logits) {
    for (long long t = blockIdx.x * (long long)NT + threadIdx.x; t < HW; t += (long long)gridDim.x * NT) {
        float a[KMD_MAX_SIZES], R[KMD_MAX_SIZES][3];
        float mb = -INFINITY;
        if (M > 1 && logits)
            for (int i = 0; i < M; ++i) mb = fmaxf(mb, __ldg(blend + i * HW + t));
        float sa = 0.f;
        for (int i = 0; i < M; ++i) {
            const float4 s = S[i * HW + t];
            R[i][0] = s.y / s.x;
            R[i][1] = s.z / s.x;
            R[i][2] = s.w / s.x;
            a[i] = M == 1 ? 1.f : (logits ? expf(__ldg(blend + i * HW + t) - mb) : __ldg(blend + i * HW + t));
            sa += a[i];
        }
        if (M > 1 && logits)
            for (int i = 0; i < M; ++i) a[i] /= sa;
        float Rh[3] = {0.f, 0.f, 0.f};
        for (int i = 0; i < M; ++i)
            for (int c = 0; c < 3; ++c) Rh[c] = fmaf(a[i], R[i][c], Rh[c]);
        const float g0 = __ldg(G + t), g1 = __ldg(G + HW + t), g2 = __ldg(G + 2 * HW + t);
        for (int i = 0; i < M; ++i) {
            if (gB) {
                float v;
                if (M == 1) v = 0.f;
                else if (logits) v = a[i] * (g0 * (R[i][0] - Rh[0]) + g1 * (R[i][1] - Rh[1]) + g2 * (R[i][2] - Rh[2]));
                else v = g0 * R[i][0] + g1 * R[i][1] + g2 * R[i][2];  // alpha given: dL/dalpha_i
                gB[i * HW + t] = v;
            }
            const float den = S[i * HW + t].x;
            const float w0 = a[i] * g0 / den, w1 = a[i] * g1 / den, w2 = a[i] * g2 / den;
            h[i * HW + t] = make_float4(w0, w1, w2, w0 * R[i][0] + w1 * R[i][1] + w2 * R[i][2]);
        }
    }
}

// 1-D transposed clamp-to-edge box along one axis (axis 0: rows, 1: columns)
__global__ void __launch_bounds__(NT) box_t(const float4* __restrict__ in, float4* __restrict__ out, int H, int W,
                                            int r, int axis) {
    const long long total = (long long)H * W;
    const int n = axis == 0 ? H : W;
    for (long long t = blockIdx.x * (long long)NT + threadIdx.x; t < total; t += (long long)gridDim.x * NT) {
        const int y = (int)(t / W), x = (int)(t - (long long)y * W);
        const int q = axis == 0 ? y : x;
        float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int p = max(q - r, 0); p <= min(q + r, n - 1); ++p) {
            // multiplicity of source p landing on q: #{o in [-r,r] : clamp(p+o) = q}
            int m;
            if (q == 0 && n > 1) m = max(0, r - p + 1);
            else if (q == n - 1 && n > 1) m = max(0, p + r - (n - 1) + 1);
            else if (n == 1) m = 2 * r + 1;
            else m = 1;
            const float4 v = axis == 0 ? in[(long long)p * W + x] : in[(long long)y * W + p];
            const float fm = (float)m;
            s.x = fmaf(fm, v.x, s.x); s.y = fmaf(fm, v.y, s.y); s.z = fmaf(fm, v.z, s.z); s.w = fmaf(fm, v.w, s.w);
        }
        out[t] = s;
    }
}

__global__ void __launch_bounds__(NT) grad_imp(const float* __restrict__ rad, const float* __restrict__ imp,
                                               const float4* __restrict__ T, float* __restrict__ gI, long long HW) {
    for (long long t = blockIdx.x * (long long)NT + threadIdx.x; t < HW; t += (long long)gridDim.x * NT) {
        const float4 v = T[t];
        const float e = expf(__ldg(imp + t));
        const float s = __ldg(rad + t) * v.x + __ldg(rad + HW + t) * v.y + __ldg(rad + 2 * HW + t) * v.z - v.w;
        gI[t] = e * s;
    }
}

}  // namespace

size_t bwd_workspace_floats(int H, int W, int M) {
    return (size_t)H * W * 4 * (2 * (size_t)M + 1);
}

cudaError_t launch_backward(const float* rad, const float* imp, const float* blend, const float* G, float* gI,
                            float* gB, int N, int H, int W, int M, const int* sizes, int logits, float* ws,
                            cudaStream_t st) {
    const long long HW = (long long)H * W;
    float4* S = reinterpret_cast<float4*>(ws);        // [M][HW]
    float4* h = S + (size_t)M * HW;                   // [M][HW]
    float4* tmp = h + (size_t)M * HW;                 // [HW]
    const int nb = blocks_for(HW);
    for (int n = 0; n < N; ++n) {
        const float* r = rad + (size_t)n * 3 * HW;
        const float* I = imp + (size_t)n * M * HW;
        for (int i = 0; i < M; ++i) {
            const int rr = (sizes[i] - 1) / 2;
            box_fwd_v<<<nb, NT, 0, st>>>(r, I + i * HW, tmp, H, W, rr);
            box_h<<<nb, NT, 0, st>>>(tmp, S + i * HW, H, W, rr);
        }
        pixel_bwd<<<nb, NT, 0, st>>>(S, blend ? blend + (size_t)n * M * HW : nullptr, G + (size_t)n * 3 * HW,
                                     gB ? gB + (size_t)n * M * HW : nullptr, h, M, HW, logits);
        for (int i = 0; i < M; ++i) {
            const int rr = (sizes[i] - 1) / 2;
            box_t<<<nb, NT, 0, st>>>(h + i * HW, tmp, H, W, rr, 0);
            box_t<<<nb, NT, 0, st>>>(tmp, h + i * HW, H, W, rr, 1);
            grad_imp<<<nb, NT, 0, st>>>(r, I + i * HW, h + i * HW, gI + ((size_t)n * M + i) * HW, HW);
        }
    }
    return cudaGetLastError();
}

}  // namespace kmd
