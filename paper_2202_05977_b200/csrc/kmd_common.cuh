// kmd_common.cuh -- shared device helpers and the kernel parameter block for
// libkmd (product path; no oracle code is included or linked here).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <utility>

// Checked builds (-DKMD_CHECKS, scripts/build_variant.sh checked -DKMD_CHECKS):
// device-side bounds / protocol assertions on every shared-memory index the
// pipelined kernels compute, trapping on a violation (compute-sanitizer is not
// available on this run's GPU pool; tests/test_gpu_checked.py runs the parity
// suite against the checked build).  Compiled out otherwise.
#ifdef KMD_CHECKS
#define KMD_CHECK(cond)                                                                              \
    do {                                                                                             \
        if (!(cond)) {                                                                               \
            printf("KMD_CHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__,  \
                   (int)blockIdx.x, (int)threadIdx.x);                                               \
            __trap();                                                                                \
        }                                                                                            \
    } while (0)
// Scheduling jitter (checked builds only): with a nonzero seed (FusedParams
// debug = env KMD_DEBUG, read once per process), every role of the TMA kernel
// sleeps a pseudo-random 0-2 us at a quarter of its protocol points (before a
// producer issue, a field job, a fusion step, a store), so the warps
// interleave differently from run to run; a missing wait or an early slot
// release then changes the output, which tests/test_gpu_checked.py compares
// bit for bit with an unperturbed run.
#define KMD_JITTER(seed, key) kmd_jitter((unsigned)(seed), (unsigned)(key))
__device__ __forceinline__ void kmd_jitter(unsigned seed, unsigned key) {
    if (seed) {
        unsigned h = (key ^ seed) * 0x9E3779B1u ^ (blockIdx.x * 0x85EBCA77u) ^ (threadIdx.x >> 5) * 0xC2B2AE3Du;
        h ^= h >> 15;
        h *= 0x2C1B3C6Du;
        h ^= h >> 12;
        if ((h & 3) == 0) __nanosleep(h >> 21);
    }
}
#else
#define KMD_CHECK(cond) \
    do {                \
    } while (0)
#define KMD_JITTER(seed, key) \
    do {                      \
    } while (0)
#endif

#include "../../include/kmd.h"

namespace kmd {

// Parameters of one fused launch.  Rows are addressed in GLOBAL frame
// coordinates so a row band (multi-GPU split) and the whole frame run the
// same arithmetic on the same pixels (bitwise band equality).
struct FusedParams {
    const float* rad;    // [N,3,buf_rows,W]
    const float* imp;    // [N,M,buf_rows,W]
    const float* blend;  // [N,M,out_rows,W] or nullptr (M == 1)
    float* out;          // [N,3,out_rows,W]
    const float* albedo; // [N,3,out_rows,W] or nullptr: out = Rhat * albedo (remodulation epilogue)
    int N, W, H;         // H = rows of the whole frame (clamp bound)
    int row_base;        // global row held by buffer row 0 of rad/imp
    int buf_rows;        // rows held by rad/imp
    int out_y0;          // global row of out/blend row 0
    int out_rows;        // rows of out/blend
    int tile_y_begin;    // global row of the first tile (multiple of the tile height)
    // tile rows of a launch: tile_rows_a rows from tile_y_begin, then (if the
    // launch has more) rows from tile_y_begin_b -- the band interior / seam
    // split (kmd_band.cu); tile_rows_a = INT_MAX for one contiguous range
    int tile_rows_a;
    int tile_y_begin_b;
    // > 0: the tile rows of this launch (else every tile row of the output);
    // set together with tile_y_begin / tile_rows_a / tile_y_begin_b
    int tile_rows_total;
    int M;               // number of maps / sizes
    int rmax;            // max_i (k_i - 1)/2
    int blend_is_logits;
    int sizes[KMD_MAX_SIZES];
    int debug;           // development switches (env KMD_DEBUG); 0 in production
    int max_ctas;        // > 0: cap on the persistent grid (to share the SMs with a concurrent launch)
    // backward pass A (kmd_bwd_tma.cu): dL/dRhat in; per size i the pair
    // (a_i / den_i, G.R_i) out through the stage buffer and tm_out
    const float* grad;   // [N,3,H,W] or nullptr
    const float* lse;    // [N,H,W] log sum_i exp(B_i) per pixel, or nullptr (pass A's softmax)
    // imp / blend hold bf16 bits (kmd_decode_filter_fuse_bf16; TMA kernel only)
    int in16;
    // "Ours MR" (Eq. 7) combine epilogue: out = f + alpha (U coarse - U D f),
    // with f this launch's fused result, coarse the combined next-coarser level
    // [N,3,H/2,W/2] and alpha [N,1,H,W] (whole frames, H and W even)
    const float* cmb_coarse;
    const float* cmb_alpha;
};

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return min(max(v, lo), hi); }

// Remodulation epilogue (Fig. 1, 258: "multiply back the albedo"):
// scales the fused value of output pixel (n, global row gy, column gx) in place.
__device__ __forceinline__ void remodulate(const FusedParams& p, int n, int gy, int gx, float& o0, float& o1,
                                           float& o2) {
    if (!p.albedo) return;
    const size_t oplane = (size_t)p.out_rows * p.W;
    const float* a = p.albedo + (size_t)n * 3 * oplane + (size_t)(gy - p.out_y0) * p.W + gx;
    o0 *= __ldg(a);
    o1 *= __ldg(a + oplane);
    o2 *= __ldg(a + 2 * oplane);
}

// ---- sm_90+/sm_100a primitives shared by the pipelined kernels -------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(b))
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* b, unsigned bytes) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(
                     smem_u32(b)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_spin(unsigned long long* b, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "SPIN_%=:\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra SPIN_%=;\n\t}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ bool mbar_test(unsigned long long* b, unsigned parity) {
    unsigned ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
    return ok != 0;
}

__device__ __forceinline__ float4 add4(float4 a, float4 b) {
    const float2 lo = __fadd2_rn(make_float2(a.x, a.y), make_float2(b.x, b.y));
    const float2 hi = __fadd2_rn(make_float2(a.z, a.w), make_float2(b.z, b.w));
    return make_float4(lo.x, lo.y, hi.x, hi.y);
}
__device__ __forceinline__ float fmin3(float a, float b, float c) {  // FMNMX3 (sm_100)
    float r;
    asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}
__device__ __forceinline__ float rcp_approx(float x) {  // MUFU.RCP, <= 1 ulp
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float ex2_approx(float x) {  // MUFU.EX2, ~2 ulp
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

}  // namespace kmd

// ---- tcgen05 tensor memory (TMEM) as per-thread staging ---------------------
// The TMA kernel keeps each field thread's radiance column in TMEM (lane =
// the thread's lane within its warp's quadrant, one 32-bit column per value):
// it is loaded from shared memory once per tile and read back by every size's
// field job, instead of 3 shared-memory loads per field pixel per size.
namespace kmd {
__device__ __forceinline__ void tmem_alloc(unsigned* smem_dst, unsigned ncols) {  // whole warp
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_dst)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(unsigned taddr, unsigned ncols) {  // whole warp
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tmem_fence_before_sync() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_fence_after_sync() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// 16 consecutive 32-bit columns of this thread's lane
__device__ __forceinline__ void tmem_st16(unsigned taddr, const float (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16};" ::"r"(taddr),
        "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
        "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15])
        : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// 4 consecutive columns; the registers are valid only after tmem_wait_ld()
__device__ __forceinline__ void tmem_ld4(unsigned taddr, float4& v) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(taddr)
                 : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// after tmem_wait_ld(): makes every later use of v depend on the wait (the
// compiler cannot hoist a use of a tcgen05.ld result above the wait)
__device__ __forceinline__ void tmem_reg_fence(float4& v) {
    asm volatile("" : "+f"(v.x), "+f"(v.y), "+f"(v.z), "+f"(v.w));
}
}  // namespace kmd
namespace kmd {
// columns c, c+1, c+2 of this thread's lane into v.x, v.y, v.z (v.w untouched);
// valid only after tmem_wait_ld()
__device__ __forceinline__ void tmem_ld3(unsigned taddr, float4& v) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];"
                 : "=f"(v.x), "=f"(v.y)
                 : "r"(taddr)
                 : "memory");
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=f"(v.z) : "r"(taddr + 2) : "memory");
}
__device__ __forceinline__ void tmem_reg_fence3(float4& v) { asm volatile("" : "+f"(v.x), "+f"(v.y), "+f"(v.z)); }
}  // namespace kmd

// ---- TMA (cp.async.bulk.tensor), bulk-group waits and the exp of the box
// sums: shared by the pipelined kernels (kmd_tma.cu, kmd_bwd_tma.cu)
namespace kmd {
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* tm, int x, int y, int z,
                                            unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
            "r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}
// L2 prefetch of a box (cp.async.bulk.prefetch.tensor): fire and forget
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* tm, int x, int y, int z) {
    asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(
                     reinterpret_cast<uint64_t>(tm)),
                 "r"(x), "r"(y), "r"(z)
                 : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* tm, int x, int y, int z, const void* src) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                     reinterpret_cast<uint64_t>(tm)),
                 "r"(x), "r"(y), "r"(z), "r"(smem_u32(src))
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// Programmatic dependent launch (KMD_PDL): a kernel launched with
// launch_pdl may start (barrier setup, tensor-map prefetch) while the previous
// kernel of the stream drains; pdl_wait() -- before the first global memory
// access -- returns once that kernel has completed and its writes are
// visible, so any producer / consumer order on the stream is kept.
#ifndef KMD_PDL
#define KMD_PDL 1
#endif
__device__ __forceinline__ void pdl_wait() {
#if KMD_PDL
    asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
__device__ __forceinline__ void pdl_launch_dependents() {
#if KMD_PDL
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
template <class... P, class... A>
inline cudaError_t launch_pdl(void (*kern)(P...), dim3 grid, dim3 threads, size_t smem, cudaStream_t st,
                              A&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = threads;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = KMD_PDL ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<A>(args)...);
}
constexpr float L2E = 1.44269502162933349609375f;        // log2(e) rounded to fp32
// exp(x) = 2^t (1 + r) with t = fl(x log2 e) and r = x - t ln 2 (one FMA with
// ln 2 rounded to fp32: the dropped t (ln 2 - fl(ln 2)) is below |t| 2^-28), to
// first order in |r| <= 2^-24 |t| ln 2.  MUFU.EX2 + 3 FP32 ops; with an exact
// 2^t this is <= 2.5 ulp for |x| <= 16 and <= 6 ulp at |x| = 88, plus
// ex2.approx's own ~2 ulp (the two-constant Cody-Waite form
// measured 2.6% slower for < 2e-7 of relative accuracy).
constexpr float LN2_HI = 0.693147182464599609375f;           // fl(ln 2)
__device__ __forceinline__ float exp_acc(float x) {
    const float t = x * L2E;
    const float r = fmaf(-t, LN2_HI, x);
    const float e = ex2_approx(t);
    return fmaf(e, r, e);
}

}  // namespace kmd
