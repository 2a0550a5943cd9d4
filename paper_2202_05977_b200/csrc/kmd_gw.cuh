// kmd_gw.cuh -- van Herk / Gil-Werman box sums along one line of float4
// values: blocks of k = 2R+1 values, window = suffix(block b) +
// prefix(block b+1), ~3 adds per output per component, only additions (no
// cancellation), in an order fixed by the window's position along the line.
// Used by the forward kernel (kmd_tma.cu) and the tiled backward (kmd_bwd.cu).
#pragma once

#include <type_traits>

#include "kmd_common.cuh"

namespace kmd {

// out[x] = sum_{j=x}^{x+2R} P[j] for x in [0, N); P produced by field(j) for
// j in [0, N + 2R), each exactly once.  Blocks of k = 2R+1 field values:
// suf = suffix sums of block b; window x = bk + t is suf[t] + prefix_{b+1}[t-1].
template <int R, int N, int B, class F, class E>
__device__ __forceinline__ void gw_block(float4 (&suf)[2 * R + 1], F& field, E& emit) {
    constexpr int K = 2 * R + 1;
    constexpr int X0 = B * K;
    if constexpr (X0 < N) {
        emit(X0, suf[0]);
        constexpr int TMAX = (K - 1 < N - 1 - X0) ? K - 1 : N - 1 - X0;  // outputs X0+1 .. X0+TMAX
        constexpr bool NEXT = X0 + K < N;
        constexpr int NROWS = NEXT ? K : TMAX;
        float4 raw[K];
#pragma unroll
        for (int t = 0; t < NROWS; ++t) raw[t] = field((B + 1) * K + t);
        float4 pre = raw[0];
#pragma unroll
        for (int t = 1; t <= TMAX; ++t) {
            if (t > 1) pre = add4(pre, raw[t - 1]);
            emit(X0 + t, add4(suf[t], pre));
        }
        if constexpr (NEXT) {
#pragma unroll
            for (int t = K - 2; t >= 0; --t) raw[t] = add4(raw[t], raw[t + 1]);
            gw_block<R, N, B + 1>(raw, field, emit);
        }
    }
}

template <int R, int N, class F, class E>
__device__ __forceinline__ void gw_line(F&& field, E&& emit) {
    constexpr int K = 2 * R + 1;
    float4 suf[K];
#pragma unroll
    for (int t = 0; t < K; ++t) suf[t] = field(t);
#pragma unroll
    for (int t = K - 2; t >= 0; --t) suf[t] = add4(suf[t], suf[t + 1]);
    gw_block<R, N, 0>(suf, field, emit);
}

// Field values base .. base+CNT-1 into dst: f1(j) one value at a time, or,
// when f1 takes (std::integral_constant<int, CNT>, float4* dst, int base), the
// whole block in one call (the TMA kernel's field: TMEM loads issued together,
// one wait).
template <int CNT, class F1>
__device__ __forceinline__ void fill_field(float4* dst, int base, F1& f1) {
    if constexpr (std::is_invocable_v<F1&, std::integral_constant<int, CNT>, float4*, int>) {
        f1(std::integral_constant<int, CNT>{}, dst, base);
    } else {
#pragma unroll
        for (int t = 0; t < CNT; ++t) dst[t] = f1(base + t);
    }
}

// The vertical (field-warp) Gil-Werman line: same sums in the same order as
// gw_line, with the block body in a rolled loop (it exists once in the code
// instead of N/K times; ~35% less field code for the paper's radii, which
// keeps the hot loop closer to the I-cache).  Measured and not kept: field
// values in pairs with packed FP32 exp (2% slower); folding the first block
// into the loop as well (another 7% less code, 5% slower); unrolling the
// block loop by 2 for every radius to drop the loop-carried MOVs (1-10%
// slower: code size; kept for R = 1 only, below).
template <int R, int N, class F1, class E>
__device__ __forceinline__ void gw_line_field(F1&& f1, E&& emit) {
    constexpr int K = 2 * R + 1;
    constexpr int NBLK = (N + K - 1) / K;
    float4 suf[K];
    fill_field<K>(suf, 0, f1);
#pragma unroll
    for (int t = K - 2; t >= 0; --t) suf[t] = add4(suf[t], suf[t + 1]);
    // blocks 0 .. NBLK-2: every output and every next-block field index is in range
    auto block = [&](int b) {
        const int x0 = b * K;
        emit(x0, suf[0]);
        float4 raw[K];
        fill_field<K>(raw, x0 + K, f1);
        float4 pre = raw[0];
#pragma unroll
        for (int t = 1; t < K; ++t) {
            if (t > 1) pre = add4(pre, raw[t - 1]);
            emit(x0 + t, add4(suf[t], pre));
        }
#pragma unroll
        for (int t = K - 2; t >= 0; --t) raw[t] = add4(raw[t], raw[t + 1]);
#pragma unroll
        for (int t = 0; t < K; ++t) suf[t] = raw[t];
    };
    // The block loop of the smallest radius (k = 3: 3-row blocks, the least
    // ILP per iteration) is unrolled by 2: measured 0.4-0.6 us faster per
    // 1080p frame; unrolling R = 2 as well (+0.7 us), R <= 3 (+3 us) or by 3-4
    // (no gain) was not.  Same operations in the same order: results unchanged.
#ifndef KMD_GW_UNROLL_RMAX
#define KMD_GW_UNROLL_RMAX 1
#endif
#ifndef KMD_GW_UNROLL_N
#define KMD_GW_UNROLL_N 2
#endif
    constexpr int kUnroll = KMD_GW_UNROLL_N;
    if constexpr (R <= KMD_GW_UNROLL_RMAX) {
#pragma unroll kUnroll
        for (int b = 0; b < NBLK - 1; ++b) block(b);
    } else {
#pragma unroll 1
        for (int b = 0; b < NBLK - 1; ++b) block(b);
    }
    // last block: outputs X0 .. N-1
    constexpr int X0 = (NBLK - 1) * K;
    constexpr int TMAX = N - 1 - X0;
    emit(X0, suf[0]);
    if constexpr (TMAX > 0) {
        float4 raw[TMAX];
        fill_field<TMAX>(raw, X0 + K, f1);
        float4 pre = raw[0];
#pragma unroll
        for (int t = 1; t <= TMAX; ++t) {
            if (t > 1) pre = add4(pre, raw[t - 1]);
            emit(X0 + t, add4(suf[t], pre));
        }
    }
}

}  // namespace kmd
