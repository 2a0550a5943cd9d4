// kmd_temporal.cu -- NEXT row 4: the temporal accumulation pre-pass of the
// paper's pipeline (§4.1: "reproject the previous frame to the
// current frame with the motion vector ... judge their geometry consistency by
// world position and shading normal ... failed pixels remain original 1 spp";
// SPEC.md:147-175 reproject / consistency_test / temporal_accumulate), fused
// into one elementwise pass.
//
// Per pixel: nearest-pixel reprojection s = floor(p + motion + 0.5) (R21), the
// fp32 consistency test with the exact operation order of include/kmd.h (the
// decision is an integer, so it is taken in the same precision and order as
// the oracle's, R22; no FMA contraction: __fmul_rn / __fadd_rn), then
// accum = mask ? (1 - a) prev_rad(s) + a cur : cur.
//
// HBM-bound (94 B/px).  Each thread owns 4 consecutive pixels of a row so the
// coalesced streams (current buffers, motion, outputs) move as 16-byte
// vectors when W % 4 == 0; the previous-frame reads are gathers (coherent for
// smooth motion), all issued together right after the reprojection.  Grid-stride over (frame, row, quad) with a grid of a few
// CTAs per SM.
#include "kmd_kernels.h"

namespace kmd {
namespace {

struct TParams {
    const float *cur_rad, *prev_rad, *prev_pos, *prev_nrm, *cur_pos, *cur_nrm, *motion;
    const unsigned char* prev_valid;
    float* accum;
    unsigned char* mask;
    int N, H, W;
    float pos_tol2, normal_tol, alpha;
};

template <bool VEC>
__device__ __forceinline__ void load4(const float* p, float (&v)[4], int cnt) {
    if (VEC) {
        const float4 t = __ldg(reinterpret_cast<const float4*>(p));
        v[0] = t.x, v[1] = t.y, v[2] = t.z, v[3] = t.w;
    } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = j < cnt ? __ldg(p + j) : 0.f;
    }
}

template <bool VEC>
__global__ void __launch_bounds__(256) temporal_kernel(const TParams t) {
    const int qw = (t.W + 3) / 4;
    const long long total = (long long)t.N * t.H * qw;
    const size_t plane = (size_t)t.H * t.W;
    for (long long it = blockIdx.x * 256LL + threadIdx.x; it < total; it += (long long)gridDim.x * 256) {
        const int q = (int)(it % qw);
        const long long ry = it / qw;
        const int y = (int)(ry % t.H), n = (int)(ry / t.H);
        const int x0 = 4 * q, cnt = min(4, t.W - x0);
        const size_t p0 = (size_t)y * t.W + x0;
        const size_t f3 = (size_t)n * 3 * plane;
        float mx[4], my[4];
        load4<VEC>(t.motion + (size_t)n * 2 * plane + p0, mx, cnt);
        load4<VEC>(t.motion + ((size_t)n * 2 + 1) * plane + p0, my, cnt);
        float cr[3][4], cp[3][4], cn[3][4];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            load4<VEC>(t.cur_rad + f3 + c * plane + p0, cr[c], cnt);
            load4<VEC>(t.cur_pos + f3 + c * plane + p0, cp[c], cnt);
            load4<VEC>(t.cur_nrm + f3 + c * plane + p0, cn[c], cnt);
        }
        // reproject all four pixels, then issue every gather at once (validity,
        // previous position / normal / radiance): one dependent load level
        // after the motion vectors instead of three
        size_t sidx[4];
        bool inb[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            // nearest pixel in fp32 (reading R21)
            const float fx = floorf(__fadd_rn(__fadd_rn((float)(x0 + j), mx[j]), 0.5f));
            const float fy = floorf(__fadd_rn(__fadd_rn((float)y, my[j]), 0.5f));
            inb[j] = j < cnt && fx >= 0.f && fx <= (float)(t.W - 1) && fy >= 0.f && fy <= (float)(t.H - 1);
            sidx[j] = inb[j] ? (size_t)(int)fy * t.W + (size_t)(int)fx : 0;
        }
        unsigned char pv[4];
        float pp[3][4], pn[3][4], pr[3][4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const size_t s = sidx[j];
            pv[j] = inb[j] ? __ldg(t.prev_valid + (size_t)n * plane + s) : 0;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                pp[c][j] = inb[j] ? __ldg(t.prev_pos + f3 + c * plane + s) : 0.f;
                pn[c][j] = inb[j] ? __ldg(t.prev_nrm + f3 + c * plane + s) : 0.f;
                pr[c][j] = inb[j] ? __ldg(t.prev_rad + f3 + c * plane + s) : 0.f;
            }
        }
        float out[3][4];
        unsigned char mk[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            bool m = inb[j] && pv[j] != 0;
            if (m) {
                // consistency test, fp32, fixed order (reading R22)
                float d[3], a[3], b[3];
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    d[c] = __fsub_rn(cp[c][j], pp[c][j]);
                    a[c] = __fsub_rn(__fmul_rn(2.f, cn[c][j]), 1.f);
                    b[c] = __fsub_rn(__fmul_rn(2.f, pn[c][j]), 1.f);
                }
                const float d2 = __fadd_rn(__fadd_rn(__fmul_rn(d[0], d[0]), __fmul_rn(d[1], d[1])), __fmul_rn(d[2], d[2]));
                const float dot = __fadd_rn(__fadd_rn(__fmul_rn(a[0], b[0]), __fmul_rn(a[1], b[1])), __fmul_rn(a[2], b[2]));
                const float aa = __fadd_rn(__fadd_rn(__fmul_rn(a[0], a[0]), __fmul_rn(a[1], a[1])), __fmul_rn(a[2], a[2]));
                const float bb = __fadd_rn(__fadd_rn(__fmul_rn(b[0], b[0]), __fmul_rn(b[1], b[1])), __fmul_rn(b[2], b[2]));
                m = d2 < t.pos_tol2 && dot > __fmul_rn(t.normal_tol, __fsqrt_rn(__fmul_rn(aa, bb)));
            }
            mk[j] = m ? 1 : 0;
#pragma unroll
            for (int c = 0; c < 3; ++c) out[c][j] = m ? fmaf(t.alpha, cr[c][j], (1.f - t.alpha) * pr[c][j]) : cr[c][j];
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            float* o = t.accum + f3 + c * plane + p0;
            if (VEC) {
                *reinterpret_cast<float4*>(o) = make_float4(out[c][0], out[c][1], out[c][2], out[c][3]);
            } else {
                for (int j = 0; j < cnt; ++j) o[j] = out[c][j];
            }
        }
        if (t.mask) {
            unsigned char* mo = t.mask + (size_t)n * plane + p0;
            if (VEC && ((reinterpret_cast<uintptr_t>(mo) & 3) == 0)) {
                *reinterpret_cast<uchar4*>(mo) = make_uchar4(mk[0], mk[1], mk[2], mk[3]);
            } else {
                for (int j = 0; j < cnt; ++j) mo[j] = mk[j];
            }
        }
    }
}

}  // namespace

cudaError_t launch_temporal(const float* cur_rad, const float* prev_rad, const float* prev_pos,
                            const float* prev_nrm, const unsigned char* prev_valid, const float* cur_pos,
                            const float* cur_nrm, const float* motion, float* accum, unsigned char* mask, int N,
                            int H, int W, float pos_tol, float normal_tol, float alpha, cudaStream_t st) {
    TParams t{cur_rad, prev_rad, prev_pos, prev_nrm, cur_pos, cur_nrm, motion, prev_valid, accum, mask,
              N, H, W, pos_tol * pos_tol, normal_tol, alpha};
    const long long total = (long long)N * H * ((W + 3) / 4);
    if (total == 0) return cudaSuccess;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const long long need = (total + 255) / 256;
    const int grid = (int)(need < (long long)sms * 8 ? need : (long long)sms * 8);
    const uintptr_t align = (uintptr_t)cur_rad | (uintptr_t)cur_pos | (uintptr_t)cur_nrm | (uintptr_t)motion |
                            (uintptr_t)accum;
    if (W % 4 == 0 && (align & 15) == 0)
        temporal_kernel<true><<<grid, 256, 0, st>>>(t);
    else
        temporal_kernel<false><<<grid, 256, 0, st>>>(t);
    return cudaGetLastError();
}

}  // namespace kmd
