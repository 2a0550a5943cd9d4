// kmd_mr.cu -- NEXT row 2: the multi-resolution "Ours MR" reconstruction
// (§5.2, Eq. 7; 324: "we fuse two filtering kernels with
// sizes 3 and 5 for each resolution"; Table 3 "Ours MR").
//
//   D = 2x2 mean downsampling, U = nearest upsampling;
//   per level l the fused kernel of kmd_tma.cu filters D^l(r);
//   o = f - alpha * U D f + alpha * U c   (Eq. 7), combined from the coarsest.
//
// Both kernels are elementwise over the FINE grid (one thread per fine pixel
// and channel, grid-stride), HBM-bound, fixed summation order.
#include "kmd_kernels.h"

namespace kmd {
namespace {

// out[n][c][y][x] = 0.25 * ((in[2y][2x] + in[2y][2x+1]) + (in[2y+1][2x] + in[2y+1][2x+1]))
// One thread per two horizontally adjacent outputs: two 16-byte loads per
// input row when the input row is 16-byte aligned (Wi % 4 == 0), else scalar.
__global__ void __launch_bounds__(256) down2_kernel(const float* __restrict__ in, float* __restrict__ out,
                                                    long long planes, int Ho, int Wo) {
    const int Wi = 2 * Wo, wp = (Wo + 1) / 2;
    const long long total = planes * Ho * wp;
    const bool vec = (Wi % 4) == 0 && ((uintptr_t)in & 15) == 0;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const long long pl = t / ((long long)Ho * wp);
        const int r = (int)(t - pl * Ho * wp), y = r / wp, x = 2 * (r - y * wp);
        const float* s = in + (pl * 2 * Ho + 2 * y) * (long long)Wi + 2 * x;
        float* o = out + (pl * Ho + y) * (long long)Wo + x;
        if (vec && x + 1 < Wo) {
            const float4 a = __ldg(reinterpret_cast<const float4*>(s));
            const float4 b = __ldg(reinterpret_cast<const float4*>(s + Wi));
            o[0] = 0.25f * ((a.x + a.y) + (b.x + b.y));
            o[1] = 0.25f * ((a.z + a.w) + (b.z + b.w));
        } else {
            for (int j = 0; j < 2 && x + j < Wo; ++j) {
                const float* q = s + 2 * j;
                o[j] = 0.25f * ((__ldg(q) + __ldg(q + 1)) + (__ldg(q + Wi) + __ldg(q + Wi + 1)));
            }
        }
    }
}

// Two pyramid levels in one pass: each thread reads a 4x4 block of the fine
// plane and writes its 2x2 block of level 1 and the level-2 pixel, each the
// 2x2 mean of the level below in the same fp32 order as down2_kernel (so the
// bits equal two down2 passes).  H0, W0 divisible by 4.
template <bool VEC>
__global__ void __launch_bounds__(256, 8) down4_kernel(const float* __restrict__ in, float* __restrict__ out1,
                                                    float* __restrict__ out2, int planes, int H2, int W2) {
    // one resident wave (launch_down4): triggering the dependent launch now
    // cannot starve this grid, and the level kernel's setup and first-tile
    // prefetch overlap the rest of it
    pdl_launch_dependents();
    const int W0 = 4 * W2, W1 = 2 * W2;
    const long long total = (long long)planes * H2 * W2;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int pl = (int)(t / ((long long)H2 * W2));
        const int r = (int)(t - (long long)pl * H2 * W2), y = r / W2, x = r - y * W2;
        const float* s = in + ((size_t)pl * 4 * H2 + 4 * y) * W0 + 4 * x;
        float v[4][4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (VEC) {
                const float4 q = __ldg(reinterpret_cast<const float4*>(s + (size_t)k * W0));
                v[k][0] = q.x, v[k][1] = q.y, v[k][2] = q.z, v[k][3] = q.w;
            } else {
                for (int m = 0; m < 4; ++m) v[k][m] = __ldg(s + (size_t)k * W0 + m);
            }
        }
        float l1[2][2];
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int b = 0; b < 2; ++b)
                l1[a][b] = 0.25f * ((v[2 * a][2 * b] + v[2 * a][2 * b + 1]) + (v[2 * a + 1][2 * b] + v[2 * a + 1][2 * b + 1]));
        float* o1 = out1 + ((size_t)pl * 2 * H2 + 2 * y) * W1 + 2 * x;
        o1[0] = l1[0][0];
        o1[1] = l1[0][1];
        o1[W1] = l1[1][0];
        o1[W1 + 1] = l1[1][1];
        out2[((size_t)pl * H2 + y) * W2 + x] = 0.25f * ((l1[0][0] + l1[0][1]) + (l1[1][0] + l1[1][1]));
    }
}

// Eq. 7: o = f - alpha * [U D f] + alpha * [U c], computed as
// fma(alpha, Uc - UDf, f).  One thread per 2x2 block of fine pixels and all
// three channels: the block's D f, the one coarse value and the 2x2 alphas are
// each read once (8-byte vectors when W is even).
template <bool VEC>
__global__ void __launch_bounds__(256) combine_kernel(const float* __restrict__ fine, const float* __restrict__ coarse,
                                                      const float* __restrict__ alpha, float* __restrict__ out,
                                                      int N, int H, int W) {
    const int Hc = H / 2, Wc = W / 2;
    const long long total = (long long)N * Hc * Wc;
    const size_t plane = (size_t)H * W, cplane = (size_t)Hc * Wc;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int n = (int)(t / ((long long)Hc * Wc));
        const int r = (int)(t - (long long)n * Hc * Wc), yc = r / Wc, xc = r - yc * Wc;
        const size_t p0 = (size_t)(2 * yc) * W + 2 * xc;
        const float* al = alpha + (size_t)n * plane + p0;
        auto ld2 = [](const float* q) {
            return VEC ? __ldg(reinterpret_cast<const float2*>(q)) : make_float2(__ldg(q), __ldg(q + 1));
        };
        auto st2 = [](float* q, float2 v) {
            if (VEC) *reinterpret_cast<float2*>(q) = v;
            else q[0] = v.x, q[1] = v.y;
        };
        const float2 a0 = ld2(al), a1 = ld2(al + W);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const float* fp = fine + ((size_t)n * 3 + c) * plane + p0;
            const float2 f0 = ld2(fp), f1 = ld2(fp + W);
            const float udf = 0.25f * ((f0.x + f0.y) + (f1.x + f1.y));
            const float d = __ldg(coarse + ((size_t)n * 3 + c) * cplane + (size_t)yc * Wc + xc) - udf;
            float* op = out + ((size_t)n * 3 + c) * plane + p0;
            st2(op, make_float2(fmaf(a0.x, d, f0.x), fmaf(a0.y, d, f0.y)));
            st2(op + W, make_float2(fmaf(a1.x, d, f1.x), fmaf(a1.y, d, f1.y)));
        }
    }
}

int grid_for(long long n) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    long long b = (n + 255) / 256;
    const long long cap = (long long)sms * 16;
    return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

}  // namespace

cudaError_t launch_down2(const float* in, float* out, long long planes, int Ho, int Wo, cudaStream_t st) {
    const long long n = planes * Ho * ((Wo + 1) / 2);
    if (n == 0) return cudaSuccess;
    down2_kernel<<<grid_for(n), 256, 0, st>>>(in, out, planes, Ho, Wo);
    return cudaGetLastError();
}

cudaError_t launch_down4(const float* in, float* out1, float* out2, int planes, int H2, int W2, cudaStream_t st) {
    const long long n = (long long)planes * H2 * W2;
    if (n == 0) return cudaSuccess;
    // at most one wave of 8 resident 256-thread CTAs per SM (grid-stride)
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int g = grid_for(n) < sms * 8 ? grid_for(n) : sms * 8;
    if (((uintptr_t)in & 15) == 0)
        down4_kernel<true><<<g, 256, 0, st>>>(in, out1, out2, planes, H2, W2);
    else
        down4_kernel<false><<<g, 256, 0, st>>>(in, out1, out2, planes, H2, W2);
    return cudaGetLastError();
}

cudaError_t launch_combine(const float* fine, const float* coarse, const float* alpha, float* out, int N, int H,
                           int W, cudaStream_t st) {
    const long long n = (long long)N * (H / 2) * (W / 2);
    if (n == 0) return cudaSuccess;
    const bool vec = (((uintptr_t)fine | (uintptr_t)alpha | (uintptr_t)out) & 7) == 0;
    if (vec) combine_kernel<true><<<grid_for(n), 256, 0, st>>>(fine, coarse, alpha, out, N, H, W);
    else combine_kernel<false><<<grid_for(n), 256, 0, st>>>(fine, coarse, alpha, out, N, H, W);
    return cudaGetLastError();
}

}  // namespace kmd
