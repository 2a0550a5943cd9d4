// kmd_direct.cu -- v1 fused decode + filter + fuse kernel ("direct separable").
//
// One CTA per 32x32 output tile of one frame.  Per kernel size k_i:
//   stage I_i (tile + r_i halo) in shared memory -> e = expf(I) once per
//   staged pixel (the "weight sharing" of Eq. 3: the weight of q is exp(I(q))
//   for every window containing q) -> premultiplied field P = (e, e r, e g, e b)
//   -> vertical k-tap sums -> horizontal k-tap sums -> R = num / den (Eq. 3+4,
//   PAPER.md:145-152; the ratio-of-box-filters form)
//   -> acc += alpha_i * R (Eq. 5).
// A tile whose importance values leave [KMD_EXP_SAFE_LO, KMD_EXP_SAFE_HI]
// (or whose radiance exceeds KMD_RADIANCE_SAFE) evaluates that size with a
// per-window max shift instead (R2/R13).
//
// Summation order is a function of the output pixel only (vertical dy = -r..r,
// then horizontal dx = -r..r), so any tiling -- including a row band on
// another GPU -- produces the same bits.
#include "kmd_common.cuh"
#include "kmd_kernels.h"

namespace kmd {

namespace {
constexpr int TW = 32, TH = 32, NT = 256, PPT = TW * TH / NT;  // pixels per thread

__global__ void __launch_bounds__(NT) fused_direct_kernel(FusedParams p) {
    extern __shared__ float4 smem4[];
    const int RW = TW + 2 * p.rmax, RH = TH + 2 * p.rmax;
    float4* P = smem4;                         // [RH*RW] premultiplied field of one size
    float4* V = P + RH * RW;                   // [TH*RW] vertical sums
    float* rad_s = reinterpret_cast<float*>(V + TH * RW);  // [3][RH*RW] radiance + r_max halo
    float* I_s = rad_s + 3 * RH * RW;          // [RH*RW] raw importance of one size
    float* alpha_s = I_s + RH * RW;            // [M][TH*TW] fusion weights

    const int n = blockIdx.z;
    const int x0 = blockIdx.x * TW;
    const int y0 = p.tile_y_begin + blockIdx.y * TH;
    const size_t bplane = (size_t)p.buf_rows * p.W;
    const size_t oplane = (size_t)p.out_rows * p.W;
    const float* rad = p.rad + (size_t)n * 3 * bplane;
    const float* imp = p.imp + (size_t)n * p.M * bplane;

    // clamp to the frame (reading R1), then into the buffer (rows a band does
    // not hold are never needed by an output it owns)
    auto brow = [&](int gy) {
        return clampi(clampi(gy, 0, p.H - 1) - p.row_base, 0, p.buf_rows - 1);
    };

    // ---- stage radiance (tile + r_max halo) ------------------------------
    bool rad_bad = false;
    for (int t = threadIdx.x; t < RH * RW; t += NT) {
        const int ry = t / RW, rx = t - ry * RW;
        const size_t off = (size_t)brow(y0 - p.rmax + ry) * p.W + clampi(x0 - p.rmax + rx, 0, p.W - 1);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const float v = __ldg(rad + c * bplane + off);
            rad_s[c * RH * RW + t] = v;
            rad_bad |= !(fabsf(v) <= KMD_RADIANCE_SAFE);
        }
    }

    // ---- fusion weights alpha_i(p) = softmax_i(B_i(p)) ----
    for (int t = threadIdx.x; t < TH * TW; t += NT) {
        const int ty = t / TW, tx = t - ty * TW;
        const int gy = y0 + ty, gx = x0 + tx;
        const bool valid = gx < p.W && gy >= p.out_y0 && gy < p.out_y0 + p.out_rows;
        if (p.M == 1 || !valid) {
            alpha_s[t] = 1.0f;
            for (int i = 1; i < p.M; ++i) alpha_s[i * TH * TW + t] = 0.0f;
            continue;
        }
        const float* b = p.blend + (size_t)n * p.M * oplane + (size_t)(gy - p.out_y0) * p.W + gx;
        if (p.blend_is_logits) {
            float beta = __ldg(b);
            for (int i = 1; i < p.M; ++i) beta = fmaxf(beta, __ldg(b + i * oplane));
            float s = 0.0f;
            for (int i = 0; i < p.M; ++i) {
                const float a = expf(__ldg(b + i * oplane) - beta);
                alpha_s[i * TH * TW + t] = a;
                s += a;
            }
            for (int i = 0; i < p.M; ++i) alpha_s[i * TH * TW + t] /= s;
        } else {
            for (int i = 0; i < p.M; ++i) alpha_s[i * TH * TW + t] = __ldg(b + i * oplane);
        }
    }

    float acc[PPT][3];
#pragma unroll
    for (int j = 0; j < PPT; ++j) acc[j][0] = acc[j][1] = acc[j][2] = 0.0f;

    for (int i = 0; i < p.M; ++i) {
        const int r = (p.sizes[i] - 1) / 2;
        const int PW = TW + 2 * r, PH = TH + 2 * r, off = p.rmax - r;
        const float* Ii = imp + (size_t)i * bplane;
        __syncthreads();  // previous size is done with I_s / P / V (and staging is visible)

        // ---- stage I_i (tile + r_i halo), range check -----------------------
        bool bad = rad_bad;
        for (int t = threadIdx.x; t < PH * PW; t += NT) {
            const int py = t / PW, px = t - py * PW;
            const float v = __ldg(Ii + (size_t)brow(y0 - r + py) * p.W + clampi(x0 - r + px, 0, p.W - 1));
            I_s[t] = v;
            bad |= !(v >= KMD_EXP_SAFE_LO && v <= KMD_EXP_SAFE_HI);
        }
        const int fallback = __syncthreads_or(bad);

        if (!fallback) {
            // e = exp(I(q)) once per staged q; P = (e, e r, e g, e b)
            for (int t = threadIdx.x; t < PH * PW; t += NT) {
                const int py = t / PW, px = t - py * PW;
                const int ridx = (py + off) * RW + px + off;
                const float e = expf(I_s[t]);
                P[t] = make_float4(e, e * rad_s[ridx], e * rad_s[RH * RW + ridx],
                                   e * rad_s[2 * RH * RW + ridx]);
            }
            __syncthreads();
            // vertical k-tap sums, dy = -r..r in order
            for (int t = threadIdx.x; t < TH * PW; t += NT) {
                const int ty = t / PW, px = t - ty * PW;
                float4 s = P[ty * PW + px];
                for (int dy = 1; dy <= 2 * r; ++dy) {
                    const float4 v = P[(ty + dy) * PW + px];
                    s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
                }
                V[t] = s;
            }
            __syncthreads();
            // horizontal k-tap sums, dx = -r..r in order; ratio; fuse
#pragma unroll
            for (int j = 0; j < PPT; ++j) {
                const int t = threadIdx.x + j * NT;
                const int ty = t / TW, tx = t - ty * TW;
                float4 s = V[ty * PW + tx];
                for (int dx = 1; dx <= 2 * r; ++dx) {
                    const float4 v = V[ty * PW + tx + dx];
                    s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
                }
                const float a = alpha_s[i * TH * TW + t];
                acc[j][0] += a * (s.y / s.x);
                acc[j][1] += a * (s.z / s.x);
                acc[j][2] += a * (s.w / s.x);
            }
        } else {
            // per-window max-shifted evaluation of Eq. 3-4 (exact rewrite, R2)
#pragma unroll 1
            for (int j = 0; j < PPT; ++j) {
                const int t = threadIdx.x + j * NT;
                const int ty = t / TW, tx = t - ty * TW;
                float m = -INFINITY;
                for (int dy = 0; dy <= 2 * r; ++dy)
                    for (int dx = 0; dx <= 2 * r; ++dx) m = fmaxf(m, I_s[(ty + dy) * PW + tx + dx]);
                float den = 0.f, n0 = 0.f, n1 = 0.f, n2 = 0.f;
                for (int dy = 0; dy <= 2 * r; ++dy)
                    for (int dx = 0; dx <= 2 * r; ++dx) {
                        const float e = expf(I_s[(ty + dy) * PW + tx + dx] - m);
                        const int ridx = (ty + dy + off) * RW + tx + dx + off;
                        den += e;
                        n0 += e * rad_s[ridx];
                        n1 += e * rad_s[RH * RW + ridx];
                        n2 += e * rad_s[2 * RH * RW + ridx];
                    }
                const float a = alpha_s[i * TH * TW + t];
                acc[j][0] += a * (n0 / den);
                acc[j][1] += a * (n1 / den);
                acc[j][2] += a * (n2 / den);
            }
        }
    }

    // ---- store the fused result ------------------------------------------
    float* out = p.out + (size_t)n * 3 * oplane;
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
        const int t = threadIdx.x + j * NT;
        const int ty = t / TW, tx = t - ty * TW;
        const int gy = y0 + ty, gx = x0 + tx;
        if (gx < p.W && gy >= p.out_y0 && gy < p.out_y0 + p.out_rows) {
            const size_t o = (size_t)(gy - p.out_y0) * p.W + gx;
            float o0 = acc[j][0], o1 = acc[j][1], o2 = acc[j][2];
            remodulate(p, n, gy, gx, o0, o1, o2);
            out[o] = o0;
            out[oplane + o] = o1;
            out[2 * oplane + o] = o2;
        }
    }
}

size_t direct_smem_bytes(int rmax, int M) {
    const int RW = TW + 2 * rmax, RH = TH + 2 * rmax;
    return sizeof(float4) * (size_t)(RH * RW + TH * RW) + sizeof(float) * (size_t)(4 * RH * RW) +
           sizeof(float) * (size_t)(M * TH * TW);
}
}  // namespace

cudaError_t launch_fused_direct(FusedParams p, cudaStream_t stream) {
    p.tile_y_begin = (p.out_y0 / TH) * TH;
    const int tiles_y = (p.out_y0 + p.out_rows - p.tile_y_begin + TH - 1) / TH;
    const dim3 grid((p.W + TW - 1) / TW, tiles_y, p.N);
    const size_t smem = direct_smem_bytes(p.rmax, p.M);
    cudaError_t err = cudaFuncSetAttribute(fused_direct_kernel,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return err;
    fused_direct_kernel<<<grid, NT, smem, stream>>>(p);
    return cudaGetLastError();
}

}  // namespace kmd
