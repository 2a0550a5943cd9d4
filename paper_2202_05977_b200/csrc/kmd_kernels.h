// kmd_kernels.h -- host-side launchers of the libkmd device kernels.
#pragma once
#include "kmd_common.cuh"

namespace kmd {

// v1: direct separable sums, one CTA per 32x32 tile (kmd_direct.cu)
cudaError_t launch_fused_direct(FusedParams p, cudaStream_t stream);

// v2: persistent warp-specialised producer/consumer kernel, k <= 13 (kmd_ws.cu)
bool ws_supported(const FusedParams& p);
cudaError_t launch_fused_ws(FusedParams p, cudaStream_t stream);

// v3: persistent warp-specialised kernel fed by TMA, k <= 13, W % 4 == 0 (kmd_tma.cu)
bool tma_supported(const FusedParams& p);
cudaError_t launch_fused_tma(FusedParams p, cudaStream_t stream);
int tma_tile_rows();  // output rows per TMA-kernel tile (the global tile grid's pitch)
// the same kernel with 28-row tiles and the Eq. 7 combine epilogue (kmd_tma_mr.cu)
int tma_mr_tile_rows();
cudaError_t launch_fused_tma_mr(FusedParams p, cudaStream_t stream);

// fusion only, Eq. 5 (kmd_fuse.cu)
cudaError_t launch_fuse_only(const float* filtered, const float* blend, float* out, int N,
                             int H, int W, int M, int blend_is_logits, cudaStream_t stream);

// albedo demodulation (op 0: x / max(albedo, eps)) and remodulation (op 1: x * albedo), kmd_fuse.cu
cudaError_t launch_albedo_op(const float* x, const float* albedo, float eps, float* out, long long n, int op,
                             cudaStream_t stream);

// multi-resolution ("Ours MR", NEXT row 2; kmd_mr.cu)
cudaError_t launch_down2(const float* in, float* out, long long planes, int Ho, int Wo, cudaStream_t st);
cudaError_t launch_down4(const float* in, float* out1, float* out2, int planes, int H2, int W2, cudaStream_t st);
cudaError_t launch_combine(const float* fine, const float* coarse, const float* alpha, float* out, int N, int H,
                           int W, cudaStream_t st);

// backward (NEXT row 3): pass A in kmd_tma.cu (h_i, G.R_i), pass B / C in
// kmd_bwd_tma.cu, the one-launch fallback in kmd_bwd.cu
cudaError_t launch_bwd_h_tma(FusedParams p, float* ws, cudaStream_t stream);
bool bwd_tma_supported(int H, int W, int M, const int* sizes, const void* a, const void* b, const void* c,
                       const void* d);
size_t bwd_tma_workspace_bytes(int N, int H, int W, int M);
cudaError_t launch_backward_tma(const float* rad, const float* imp, const float* blend, const float* G, float* gI,
                                float* gB, int N, int H, int W, int M, const int* sizes, int logits, void* ws,
                                cudaStream_t st);
size_t bwd_workspace_floats(int H, int W, int M);
cudaError_t launch_backward(const float* rad, const float* imp, const float* blend, const float* G, float* gI,
                            float* gB, int N, int H, int W, int M, const int* sizes, int logits, float* ws,
                            cudaStream_t st);

// temporal accumulation pre-pass (NEXT row 4; kmd_temporal.cu)
cudaError_t launch_temporal(const float* cur_rad, const float* prev_rad, const float* prev_pos,
                            const float* prev_nrm, const unsigned char* prev_valid, const float* cur_pos,
                            const float* cur_nrm, const float* motion, float* accum, unsigned char* mask, int N,
                            int H, int W, float pos_tol, float normal_tol, float alpha, cudaStream_t st);

// error detail for kmd_last_error() from any translation unit (kmd_api.cu)
kmd_status api_fail(kmd_status s, const char* fmt, ...);
void api_clear_error();

// kernel variant of the last fused launch on this host thread (kmd_last_kernel)
enum LastKernel { LK_NONE = 0, LK_DIRECT = 1, LK_WS = 2, LK_TMA = 3, LK_BWD_TILE = 10, LK_BWD_TMA = 11, LK_TMA_SPEC = 100,
                  LK_TMA_SPEC_ALB = 150, LK_TMA_BF16 = 200, LK_TMA_MR = 300, LK_TMA_MR_CMB = 301 };
void set_last_kernel(int k);

}  // namespace kmd
