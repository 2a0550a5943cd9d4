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

// out[n][c][y][x] = 0.25 * (in[2y][2x] + in[2y][2x+1] + in[2y+1][2x] + in[2y+1][2x+1])
__global__ void __launch_bounds__(256) down2_kernel(const float* __restrict__ in, float* __restrict__ out,
                                                    long long planes, int Ho, int Wo) {
    const long long total = planes * Ho * Wo;
    const int Wi = 2 * Wo;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const long long pl = t / ((long long)Ho * Wo);
        const int r = (int)(t - pl * Ho * Wo), y = r / Wo, x = r - y * Wo;
        const float* s = in + (pl * 2 * Ho + 2 * y) * (long long)Wi + 2 * x;
        const float a = __ldg(s), b = __ldg(s + 1), c = __ldg(s + Wi), d = __ldg(s + Wi + 1);
        out[t] = 0.25f * ((a + b) + (c + d));
    }
}

// Eq. 7: o = f - alpha * [U D f] + alpha * [U c]
__global__ void __launch_bounds__(256) combine_kernel(const float* __restrict__ fine, const float* __restrict__ coarse,
                                                      const float* __restrict__ alpha, float* __restrict__ out,
                                                      int N, int H, int W) {
    const long long total = (long long)N * 3 * H * W;
    const int Hc = H / 2, Wc = W / 2;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const long long plane = t / ((long long)H * W);  // n*3 + c
        const int r = (int)(t - plane * H * W), y = r / W, x = r - y * W;
        const long long n = plane / 3;
        const float* fp = fine + plane * H * W;
        const int y0 = y & ~1, x0 = x & ~1;
        const float a = __ldg(fp + (long long)y0 * W + x0), b = __ldg(fp + (long long)y0 * W + x0 + 1);
        const float c = __ldg(fp + (long long)(y0 + 1) * W + x0), d = __ldg(fp + (long long)(y0 + 1) * W + x0 + 1);
        const float udf = 0.25f * ((a + b) + (c + d));
        const float uc = __ldg(coarse + plane * Hc * Wc + (long long)(y >> 1) * Wc + (x >> 1));
        const float al = __ldg(alpha + n * H * W + (long long)y * W + x);
        const float f = __ldg(fp + (long long)y * W + x);
        out[t] = fmaf(al, uc - udf, f);
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
    const long long n = planes * Ho * Wo;
    if (n == 0) return cudaSuccess;
    down2_kernel<<<grid_for(n), 256, 0, st>>>(in, out, planes, Ho, Wo);
    return cudaGetLastError();
}

cudaError_t launch_combine(const float* fine, const float* coarse, const float* alpha, float* out, int N, int H,
                           int W, cudaStream_t st) {
    const long long n = (long long)N * 3 * H * W;
    if (n == 0) return cudaSuccess;
    combine_kernel<<<grid_for(n), 256, 0, st>>>(fine, coarse, alpha, out, N, H, W);
    return cudaGetLastError();
}

}  // namespace kmd
