// kmd_band.cu -- multi-GPU row bands (BASELINE configs[3]):
// the NCCL halo exchange and the band step that overlaps it with the band
// interior.  Declared in include/kmd.h.
//
// Every output pixel of Eq. 3-5 depends only on its (2 r_max + 1)^2
// neighbourhood, so a frame cut into row bands needs one
// exchange step per frame: r_max rows of the 3 radiance planes and the M
// importance planes from each neighbour (the fusion logits need none).  One
// grouped NCCL call moves every plane's halo rows; the interior tile rows,
// which read owned rows only, run on the compute stream meanwhile, and the
// seam tile rows follow once the exchange has landed.
//
// NCCL is loaded at run time (dlopen "libnccl.so.2"): in a process that
// imported torch this resolves to torch's already-loaded NCCL, so libkmd and
// torch.distributed share one NCCL; the rest of libkmd never needs it.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdio>
#include <cstring>
#include <mutex>
#include <type_traits>
#include <vector>

#include "kmd_kernels.h"

namespace {

struct NcclApi {
    bool ok = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
    ncclResult_t (*CommUserRank)(const ncclComm_t, int*) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    char why[256] = "";
};

NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            snprintf(api.why, sizeof(api.why), "dlopen libnccl.so.2: %s", dlerror());
            return;
        }
        bool all = true;
        auto sym = [&](auto& fn, const char* name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
            if (!fn) {
                all = false;
                snprintf(api.why, sizeof(api.why), "libnccl.so.2 lacks %s", name);
            }
        };
        sym(api.GetUniqueId, "ncclGetUniqueId");
        sym(api.CommInitRank, "ncclCommInitRank");
        sym(api.CommDestroy, "ncclCommDestroy");
        sym(api.GroupStart, "ncclGroupStart");
        sym(api.GroupEnd, "ncclGroupEnd");
        sym(api.Send, "ncclSend");
        sym(api.Recv, "ncclRecv");
        sym(api.CommCount, "ncclCommCount");
        sym(api.CommUserRank, "ncclCommUserRank");
        sym(api.GetErrorString, "ncclGetErrorString");
        api.ok = all;
    });
    return api;
}

kmd_status nccl_fail(ncclResult_t r, const char* what) {
    return kmd::api_fail(KMD_ERR_NCCL, "%s: %s", what, nccl().GetErrorString ? nccl().GetErrorString(r) : "?");
}

kmd_status need_nccl() {
    if (!nccl().ok) return kmd::api_fail(KMD_ERR_NCCL, "NCCL unavailable (%s)", nccl().why);
    return KMD_OK;
}

// library-owned events of the band step (per host thread and device, created once)
struct BandEvents {
    cudaEvent_t ready = nullptr, exchanged = nullptr;
    int dev = -1;
};
thread_local BandEvents g_be;

cudaError_t band_events(BandEvents** out) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (g_be.dev != dev) {
        BandEvents b;
        if ((e = cudaEventCreateWithFlags(&b.ready, cudaEventDisableTiming)) != cudaSuccess) return e;
        if ((e = cudaEventCreateWithFlags(&b.exchanged, cudaEventDisableTiming)) != cudaSuccess) return e;
        b.dev = dev;
        g_be = b;
    }
    *out = &g_be;
    return cudaSuccess;
}

thread_local std::vector<float*> g_planes;  // host array of plane pointers, reused across calls

}  // namespace

extern "C" {

kmd_status kmd_nccl_unique_id(uint8_t id[KMD_NCCL_ID_BYTES]) {
    kmd::api_clear_error();
    static_assert(sizeof(ncclUniqueId) == KMD_NCCL_ID_BYTES, "ncclUniqueId is 128 bytes");
    if (!id) return kmd::api_fail(KMD_ERR_NULL, "id is NULL");
    if (kmd_status s = need_nccl()) return s;
    ncclUniqueId u;
    ncclResult_t r = nccl().GetUniqueId(&u);
    if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
    memcpy(id, &u, sizeof(u));
    return KMD_OK;
}

kmd_status kmd_comm_init(void** comm, const uint8_t id[KMD_NCCL_ID_BYTES], int32_t nranks, int32_t rank) {
    kmd::api_clear_error();
    if (!comm || !id) return kmd::api_fail(KMD_ERR_NULL, "comm or id is NULL");
    if (nranks < 1 || rank < 0 || rank >= nranks)
        return kmd::api_fail(KMD_ERR_DIM, "rank %d of %d ranks", rank, nranks);
    if (kmd_status s = need_nccl()) return s;
    ncclUniqueId u;
    memcpy(&u, id, sizeof(u));
    ncclComm_t c = nullptr;
    ncclResult_t r = nccl().CommInitRank(&c, nranks, u, rank);
    if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitRank");
    *comm = c;
    return KMD_OK;
}

kmd_status kmd_comm_destroy(void* comm) {
    kmd::api_clear_error();
    if (!comm) return KMD_OK;
    if (kmd_status s = need_nccl()) return s;
    ncclResult_t r = nccl().CommDestroy((ncclComm_t)comm);
    if (r != ncclSuccess) return nccl_fail(r, "ncclCommDestroy");
    return KMD_OK;
}

kmd_status kmd_halo_exchange(void* comm, float* const* planes, int32_t n_planes, int32_t band_rows,
                             int32_t W, int32_t halo, int32_t peer_up, int32_t peer_down,
                             kmd_stream_t stream) {
    kmd::api_clear_error();
    if (n_planes < 0 || band_rows < 1 || W < 1 || halo < 0 || halo > band_rows)
        return kmd::api_fail(KMD_ERR_DIM, "n_planes=%d band_rows=%d W=%d halo=%d (need band_rows >= halo >= 0)",
                             n_planes, band_rows, W, halo);
    if (peer_up < -1 || peer_down < -1) return kmd::api_fail(KMD_ERR_DIM, "peer ranks must be >= -1");
    const bool up = peer_up >= 0 && halo > 0, down = peer_down >= 0 && halo > 0;
    if (n_planes == 0 || (!up && !down)) return KMD_OK;
    if (!comm || !planes) return kmd::api_fail(KMD_ERR_NULL, "comm or planes is NULL");
    if (kmd_status s = need_nccl()) return s;
    int nranks = 0;
    ncclResult_t r = nccl().CommCount((ncclComm_t)comm, &nranks);
    if (r != ncclSuccess) return nccl_fail(r, "ncclCommCount");
    if (peer_up >= nranks || peer_down >= nranks)
        return kmd::api_fail(KMD_ERR_DIM, "peer (%d, %d) outside a communicator of %d ranks", peer_up, peer_down,
                             nranks);
    for (int p = 0; p < n_planes; ++p)
        if (!planes[p]) return kmd::api_fail(KMD_ERR_NULL, "planes[%d] is NULL", p);
    const int top = up ? halo : 0;
    const size_t rowsz = (size_t)W, blk = (size_t)halo * W;
    cudaStream_t st = (cudaStream_t)stream;
    ncclComm_t c = (ncclComm_t)comm;
    NcclApi& n = nccl();
    if ((r = n.GroupStart()) != ncclSuccess) return nccl_fail(r, "ncclGroupStart");
    ncclResult_t bad = ncclSuccess;
    for (int p = 0; p < n_planes && bad == ncclSuccess; ++p) {
        float* base = planes[p];
        // per plane: recv from up, recv from down, send to up, send to down
        if (up) bad = n.Recv(base, blk, ncclFloat32, peer_up, c, st);
        if (down && bad == ncclSuccess) bad = n.Recv(base + (size_t)(top + band_rows) * rowsz, blk, ncclFloat32, peer_down, c, st);
        if (up && bad == ncclSuccess) bad = n.Send(base + (size_t)top * rowsz, blk, ncclFloat32, peer_up, c, st);
        if (down && bad == ncclSuccess)
            bad = n.Send(base + (size_t)(top + band_rows - halo) * rowsz, blk, ncclFloat32, peer_down, c, st);
    }
    r = n.GroupEnd();
    if (bad != ncclSuccess) return nccl_fail(bad, "ncclSend/ncclRecv");
    if (r != ncclSuccess) return nccl_fail(r, "ncclGroupEnd");
    return KMD_OK;
}

kmd_status kmd_band_step(void* comm, float* radiance, float* importance, const float* blend, float* out,
                         int32_t N, int32_t band_rows, int32_t W, int32_t halo, int32_t peer_up,
                         int32_t peer_down, int32_t y0, int32_t H_global, const kmd_config* cfg,
                         kmd_stream_t stream, kmd_stream_t comm_stream) {
    kmd::api_clear_error();
    if (!cfg) return kmd::api_fail(KMD_ERR_NULL, "cfg is NULL");
    if (halo < 0 || N < 0) return kmd::api_fail(KMD_ERR_DIM, "halo=%d, N=%d must be >= 0", halo, N);
    const int top = peer_up >= 0 ? halo : 0, bot = peer_down >= 0 ? halo : 0;
    // validate the band (and take the N == 0 no-op) before touching NCCL or streams
    kmd_status s = kmd_decode_filter_fuse_band_part(radiance, importance, blend, out, 0, band_rows, W, top, bot, y0,
                                                    H_global, cfg, KMD_BAND_ALL, stream);
    if (s) return s;
    if (N == 0) return KMD_OK;
    const bool exchange = (top > 0 || bot > 0);
    cudaStream_t st = (cudaStream_t)stream, cst = comm_stream ? (cudaStream_t)comm_stream : st;
    if (exchange) {
        if (!comm) return kmd::api_fail(KMD_ERR_NULL, "comm is NULL with a neighbour (peers %d, %d)", peer_up, peer_down);
        const int M = cfg->num_sizes;
        const size_t plane = (size_t)(top + band_rows + bot) * W;
        g_planes.clear();
        for (int n = 0; n < N; ++n) {
            for (int c = 0; c < 3; ++c) g_planes.push_back(radiance + ((size_t)n * 3 + c) * plane);
            for (int i = 0; i < M; ++i) g_planes.push_back(importance + ((size_t)n * M + i) * plane);
        }
        BandEvents* ev = nullptr;
        cudaError_t e = band_events(&ev);
        if (e != cudaSuccess) return kmd::api_fail(KMD_ERR_CUDA, "band events: %s", cudaGetErrorString(e));
        if (cst != st) {
            // the owned rows are produced on `stream`: the exchange starts after them
            if ((e = cudaEventRecord(ev->ready, st)) != cudaSuccess || (e = cudaStreamWaitEvent(cst, ev->ready, 0)) != cudaSuccess)
                return kmd::api_fail(KMD_ERR_CUDA, "band step fork: %s", cudaGetErrorString(e));
        }
        s = kmd_halo_exchange(comm, g_planes.data(), (int32_t)g_planes.size(), band_rows, W, halo, peer_up, peer_down,
                              cst);
        if (s) return s;
        if (cst != st) {
            if ((e = cudaEventRecord(ev->exchanged, cst)) != cudaSuccess)
                return kmd::api_fail(KMD_ERR_CUDA, "band step event: %s", cudaGetErrorString(e));
            // interior tile rows: owned rows only, concurrent with the exchange
            s = kmd_decode_filter_fuse_band_part(radiance, importance, blend, out, N, band_rows, W, top, bot, y0,
                                                 H_global, cfg, KMD_BAND_INTERIOR, stream);
            if (s) return s;
            if ((e = cudaStreamWaitEvent(st, ev->exchanged, 0)) != cudaSuccess)
                return kmd::api_fail(KMD_ERR_CUDA, "band step join: %s", cudaGetErrorString(e));
            return kmd_decode_filter_fuse_band_part(radiance, importance, blend, out, N, band_rows, W, top, bot, y0,
                                                    H_global, cfg, KMD_BAND_SEAMS, stream);
        }
    }
    return kmd_decode_filter_fuse_band_part(radiance, importance, blend, out, N, band_rows, W, top, bot, y0, H_global,
                                            cfg, KMD_BAND_ALL, stream);
}

}  // extern "C"
