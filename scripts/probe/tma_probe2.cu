// TMA probe 2: which bulk-copy forms work on this box?
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(unsigned long long* b) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(b)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void bar_expect(unsigned long long* b, unsigned bytes) {
    asm volatile("{ .reg .b64 st; mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1; }" ::"r"(su32(b)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bar_wait(unsigned long long* b) {
    asm volatile("{ .reg .pred p; W_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W_%=; }" ::"r"(
                     su32(b))
                 : "memory");
}

// mode 0: 1D bulk copy; 1: 2D tensor; 2: 3D tensor; 3: 3D tensor, coords >= 0
__global__ void probe2(int mode, int cx, int cy, const __grid_constant__ CUtensorMap tm2, const __grid_constant__ CUtensorMap tm3,
                       const float* src, float* out) {
    __shared__ __align__(1024) float buf[36 * 64];
    __shared__ __align__(8) unsigned long long bar;
    if (threadIdx.x == 0) bar_init(&bar);
    __syncthreads();
    if (threadIdx.x == 0) {
        bar_expect(&bar, mode == 0 ? 64 * 4 : 36 * 64 * 4);
        if (mode == 4) {
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
                "[%5];" ::"r"(su32(buf)),
                "l"((uint64_t)&tm3), "r"(0), "r"(0), "r"(0), "r"(su32(&bar))
                : "memory");
        } else if (mode == 0) {
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             su32(buf)),
                         "l"((uint64_t)src), "r"(256), "r"(su32(&bar))
                         : "memory");
        } else if (mode == 1) {
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
                    "r"(su32(buf)),
                "l"((uint64_t)&tm2), "r"(cx), "r"(cy), "r"(su32(&bar))
                : "memory");
        } else {
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
                "[%5];" ::"r"(su32(buf)),
                "l"((uint64_t)&tm3), "r"(cx), "r"(cy), "r"(0), "r"(su32(&bar))
                : "memory");
        }
    }
    bar_wait(&bar);
    if (mode == 4) {
        __syncthreads();
        for (int i = threadIdx.x; i < 36 * 64; i += blockDim.x) buf[i] = 1.0f;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
            asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                             (uint64_t)&tm3), "r"(cx), "r"(cy), "r"(0), "r"(su32(buf)) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        }
        return;
    }
    float s = 0;
    const int n = mode == 0 ? 64 : 36 * 64;
    for (int i = threadIdx.x; i < n; i += blockDim.x) s += buf[i];
    atomicAdd(out, s);
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

extern "C" int run_probe2(int mode, int cx, int cy, int l2, const float* src, int W, int H, float* out) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess) return -1;
    EncodeFn enc = (EncodeFn)f;
    CUtensorMap tm2, tm3;
    cuuint64_t d2[2] = {(cuuint64_t)W, (cuuint64_t)H}, s2[1] = {(cuuint64_t)W * 4};
    cuuint32_t b2[2] = {64, 36}, e2[2] = {1, 1};
    CUresult r = enc(&tm2, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)src, d2, s2, b2, e2, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("enc2=%d ", (int)r);
    cuuint64_t d3[3] = {(cuuint64_t)W, (cuuint64_t)H, 1}, s3[2] = {(cuuint64_t)W * 4, (cuuint64_t)W * 4 * H};
    cuuint32_t b3[3] = {64, 36, 1}, e3[3] = {1, 1, 1};
    r = enc(&tm3, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)src, d3, s3, b3, e3, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, l2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("enc3=%d q=%d ", (int)r, (int)q);
    if (0) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(1);
        cfg.blockDim = dim3(128);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 1;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaError_t le = cudaLaunchKernelEx(&cfg, probe2, mode, cx, cy, tm2, tm3, src, out);
        printf("launchEx=%d ", (int)le);
    } else {
        probe2<<<1, 128>>>(mode, cx, cy, tm2, tm3, src, out);
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("sync=%s\n", cudaGetErrorString(e));
    fflush(stdout);
    return e == cudaSuccess ? 0 : -3;
}
