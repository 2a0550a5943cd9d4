// Minimal TMA probe: one 2D/3D tile load into smem, mbarrier expect_tx, checksum.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int VARIANT>
__global__ void probe(const __grid_constant__ CUtensorMap tm_param, const CUtensorMap* tm_global, float* out) {
    const CUtensorMap& tm = (VARIANT & 4) ? *tm_global : tm_param;
    __shared__ __align__(1024) float buf[36 * 64];
    __shared__ __align__(8) unsigned long long bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        if (VARIANT & 1) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (VARIANT & 2) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("{ .reg .b64 st; mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1; }" ::"r"(su32(&bar)),
                     "r"(36 * 64 * 4) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
                "r"(su32(buf)), "l"((uint64_t)&tm), "r"(-6), "r"(-6), "r"(0), "r"(su32(&bar))
            : "memory");
    }
    asm volatile("{ .reg .pred p; W_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W_%=; }" ::"r"(
                     su32(&bar))
                 : "memory");
    float s = 0;
    for (int i = threadIdx.x; i < 36 * 64; i += blockDim.x) s += buf[i];
    atomicAdd(out, s);
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

extern "C" int run_probe(int variant, const float* src, int W, int H, float* out) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess) return -1;
    CUtensorMap tm;
    cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, 1};
    cuuint64_t str[2] = {(cuuint64_t)W * 4, (cuuint64_t)W * 4 * H};
    cuuint32_t box[3] = {64, 36, 1}, es[3] = {1, 1, 1};
    CUresult r = ((EncodeFn)f)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)src, dims, str, box, es,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return -2;
    unsigned char* hb = (unsigned char*)&tm;
    printf("desc:"); for (int i = 0; i < 32; ++i) printf(" %02x", hb[i]); printf("\n");
    CUtensorMap* dtm = nullptr;
    cudaMalloc(&dtm, sizeof(CUtensorMap));
    cudaMemcpy(dtm, &tm, sizeof(CUtensorMap), cudaMemcpyHostToDevice);
    switch (variant) {
        case 0: probe<0><<<1, 128>>>(tm, dtm, out); break;
        case 1: probe<1><<<1, 128>>>(tm, dtm, out); break;
        case 4: probe<4><<<1, 128>>>(tm, dtm, out); break;
        default: probe<5><<<1, 128>>>(tm, dtm, out); break;
    }
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("cuda error: %s\n", cudaGetErrorString(e)); fflush(stdout); return -3; }
    return 0;
}
