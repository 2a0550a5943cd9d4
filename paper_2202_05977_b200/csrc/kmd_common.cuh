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
};

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return min(max(v, lo), hi); }

}  // namespace kmd
