// TMA streaming probe: one elected thread per CTA streams [rows][68]-float boxes
// (like the importance boxes of kmd_tma.cu) through an NS-deep smem ring; a
// consumer warp waits for each box and releases it at once.  Measures the
// achievable HBM->SM rate vs ring depth / box size.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(unsigned long long* b, unsigned c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void bar_expect(unsigned long long* b, unsigned bytes) {
    asm volatile("{ .reg .b64 st; mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1; }" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_arrive(unsigned long long* b) {
    asm volatile("{ .reg .b64 st; mbarrier.arrive.shared::cta.b64 st, [%0]; }" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(unsigned long long* b, unsigned par) {
    asm volatile("{ .reg .pred p; W_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W_%=; }" ::"r"(su32(b)), "r"(par) : "memory");
}

__global__ void stream_kernel(const __grid_constant__ CUtensorMap tm, int ns, int rows, int W, int H, int planes, float* sink) {
    extern __shared__ __align__(1024) unsigned char smem[];
    const int box_bytes = (rows * 68 * 4 + 127) / 128 * 128;
    unsigned long long* full = reinterpret_cast<unsigned long long*>(smem + ns * box_bytes);
    unsigned long long* empty = full + ns;
    if (threadIdx.x == 0) {
        for (int s = 0; s < ns; ++s) { bar_init(&full[s], 1); bar_init(&empty[s], 1); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int tiles_x = (W + 51) / 52, tiles_y = (H + rows - 13) / (rows - 12);
    const int ntiles = tiles_x * tiles_y * planes;
    const int my = ntiles > (int)blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    if (threadIdx.x == 0) {
        for (int k = 0; k < my; ++k) {
            const int t = blockIdx.x + k * gridDim.x;
            const int pl = t / (tiles_x * tiles_y), r = t % (tiles_x * tiles_y);
            const int ty = r / tiles_x, tx = r % tiles_x;
            const int s = k % ns;
            bar_wait(&empty[s], ((k / ns) & 1) ^ 1);
            bar_expect(&full[s], rows * 68 * 4);
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                         ::"r"(su32(smem + s * box_bytes)), "l"((uint64_t)&tm), "r"(tx * 52 - 8), "r"(ty * (rows - 12) - 6), "r"(pl),
                           "r"(su32(&full[s])) : "memory");
        }
    } else if (threadIdx.x == 32) {
        float acc = 0;
        for (int k = 0; k < my; ++k) {
            const int s = k % ns;
            bar_wait(&full[s], (k / ns) & 1);
            acc += reinterpret_cast<float*>(smem + s * box_bytes)[k & 63];
            bar_arrive(&empty[s]);
        }
        if (acc == 12345.f) *sink = acc;
    }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

extern "C" float run_stream(const float* src, int W, int H, int planes, int ns, int rows, int ctas_per_sm, float* sink) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
    CUtensorMap tm;
    cuuint64_t d[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)planes}, st[2] = {(cuuint64_t)W * 4, (cuuint64_t)W * 4 * H};
    cuuint32_t box[3] = {68, (cuuint32_t)rows, 1}, es[3] = {1, 1, 1};
    ((EncodeFn)f)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)src, d, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const size_t smem = (size_t)ns * ((rows * 68 * 4 + 127) / 128 * 128) + 2 * ns * 8 + 64;
    cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int grid = 148 * ctas_per_sm;
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int w = 0; w < 3; ++w) stream_kernel<<<grid, 64, smem>>>(tm, ns, rows, W, H, planes, sink);
    cudaEventRecord(a);
    const int iters = 10;
    for (int w = 0; w < iters; ++w) stream_kernel<<<grid, 64, smem>>>(tm, ns, rows, W, H, planes, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return -1; }
    return ms / iters;
}
