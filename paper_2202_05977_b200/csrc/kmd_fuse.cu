// kmd_fuse.cu -- Eq. 5 on its own:
//   Rhat(p,c) = sum_i alpha_i(p) R^{k_i}(p,c),  alpha = softmax_i(B_i(p)).
// Elementwise over pixels; HBM-bound (4*(3M + M + 3) bytes per pixel).
#include "kmd_kernels.h"

namespace kmd {
namespace {

__global__ void __launch_bounds__(256) fuse_kernel(const float* __restrict__ filtered,
                                                   const float* __restrict__ blend,
                                                   float* __restrict__ out, int N, long long HW,
                                                   int M, int blend_is_logits) {
    const long long total = (long long)N * HW;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const long long n = t / HW, q = t - n * HW;
        const float* f = filtered + n * M * 3 * HW + q;
        const float* b = blend ? blend + n * M * HW + q : nullptr;
        float a[KMD_MAX_SIZES];
        if (M == 1) {
            a[0] = 1.0f;
        } else if (blend_is_logits) {
            float beta = __ldg(b);
            for (int i = 1; i < M; ++i) beta = fmaxf(beta, __ldg(b + i * HW));
            float s = 0.f;
            for (int i = 0; i < M; ++i) {
                a[i] = expf(__ldg(b + i * HW) - beta);
                s += a[i];
            }
            for (int i = 0; i < M; ++i) a[i] /= s;
        } else {
            for (int i = 0; i < M; ++i) a[i] = __ldg(b + i * HW);
        }
        float o0 = 0.f, o1 = 0.f, o2 = 0.f;
        for (int i = 0; i < M; ++i) {
            o0 += a[i] * __ldg(f + (i * 3 + 0) * HW);
            o1 += a[i] * __ldg(f + (i * 3 + 1) * HW);
            o2 += a[i] * __ldg(f + (i * 3 + 2) * HW);
        }
        float* o = out + n * 3 * HW + q;
        o[0] = o0;
        o[HW] = o1;
        o[2 * HW] = o2;
    }
}

// irradiance = radiance / max(albedo, eps);
// remodulation multiplies back.  Elementwise, HBM-bound, float4 when aligned.
__global__ void __launch_bounds__(256) albedo_kernel(const float* __restrict__ x, const float* __restrict__ a,
                                                     float eps, float* __restrict__ out, long long n, int op) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
         t += (long long)gridDim.x * blockDim.x) {
        const float v = __ldg(x + t), al = __ldg(a + t);
        out[t] = op == 0 ? v / fmaxf(al, eps) : v * al;
    }
}

}  // namespace

cudaError_t launch_albedo_op(const float* x, const float* albedo, float eps, float* out, long long n, int op,
                             cudaStream_t stream) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    long long blocks = (n + 255) / 256;
    if (blocks > (long long)sms * 16) blocks = (long long)sms * 16;
    if (blocks < 1) blocks = 1;
    albedo_kernel<<<(unsigned)blocks, 256, 0, stream>>>(x, albedo, eps, out, n, op);
    return cudaGetLastError();
}

cudaError_t launch_fuse_only(const float* filtered, const float* blend, float* out, int N,
                             int H, int W, int M, int blend_is_logits, cudaStream_t stream) {
    const long long HW = (long long)H * W;
    const long long total = (long long)N * HW;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    long long blocks = (total + 255) / 256;
    const long long cap = (long long)sms * 8;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    fuse_kernel<<<(unsigned)blocks, 256, 0, stream>>>(filtered, blend, out, N, HW, M,
                                                      blend_is_logits);
    return cudaGetLastError();
}

}  // namespace kmd
