// kmd_common.cuh -- shared device helpers and the kernel parameter block for
// libkmd (product path; no oracle code is included or linked here).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

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
