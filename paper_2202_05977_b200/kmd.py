"""Thin Python binding of libkmd (include/kmd.h): argument marshalling only.

Every step of the reconstruction runs in libkmd's CUDA kernels; this module
checks tensor dtype/device/shape/contiguity, passes ``data_ptr()``s and the
current CUDA stream, and turns a non-zero ``kmd_status`` into ``KmdError``.
There is no CPU fallback: if libkmd.so is missing or fails to load, every call
raises.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import torch

from . import _build

_HERE = os.path.dirname(os.path.abspath(__file__))
# KMD_LIB selects another build of the same library (e.g. libkmd_checked.so,
# the -DKMD_CHECKS build with device-side bounds assertions)
LIB_PATH = os.environ.get("KMD_LIB") or os.path.join(_HERE, "libkmd.so")

KMD_MAX_SIZES = 8
KMD_MAX_K = 31
STATUS = {0: "KMD_OK", 1: "KMD_ERR_NULL", 2: "KMD_ERR_CONFIG", 3: "KMD_ERR_DIM",
          4: "KMD_ERR_ALIGN", 5: "KMD_ERR_ALIAS", 6: "KMD_ERR_CUDA", 7: "KMD_ERR_NCCL"}


class KmdError(RuntimeError):
    def __init__(self, status: int, detail: str):
        self.status = status
        self.name = STATUS.get(status, f"status {status}")
        super().__init__(f"{self.name}: {detail}")


class kmd_config(ctypes.Structure):
    _fields_ = [("num_sizes", ctypes.c_int32),
                ("sizes", ctypes.c_int32 * KMD_MAX_SIZES),
                ("blend_is_logits", ctypes.c_int32),
                ("border", ctypes.c_int32)]


def make_config(sizes: Sequence[int], blend_is_logits: bool = True) -> kmd_config:
    cfg = kmd_config()
    cfg.num_sizes = len(sizes)
    for i, k in enumerate(list(sizes)[:KMD_MAX_SIZES]):
        cfg.sizes[i] = int(k)
    cfg.blend_is_logits = int(bool(blend_is_logits))
    cfg.border = 0
    return cfg


KMD_MR_MAX_LEVELS = 4


class kmd_mr_config(ctypes.Structure):
    _fields_ = [("levels", ctypes.c_int32), ("level", kmd_config * KMD_MR_MAX_LEVELS)]


def make_mr_config(sizes_per_level: Sequence[Sequence[int]]) -> kmd_mr_config:
    cfg = kmd_mr_config()
    cfg.levels = len(sizes_per_level)
    for l, sz in enumerate(list(sizes_per_level)[:KMD_MR_MAX_LEVELS]):
        cfg.level[l] = make_config(sz)
    return cfg


_lib = None

EXPORTS = ("kmd_decode_filter_fuse", "kmd_decode_filter_fuse_bf16", "kmd_decode_filter_fuse_remod",
           "kmd_demodulate",
           "kmd_mr_workspace_bytes", "kmd_mr_decode_filter_fuse", "kmd_downsample2x2",
           "kmd_combine_resolutions", "kmd_backward_workspace_bytes",
           "kmd_decode_filter_fuse_backward", "kmd_temporal_accumulate",
           "kmd_remodulate", "kmd_decode_filter", "kmd_fuse",
           "kmd_decode_filter_fuse_band", "kmd_decode_filter_fuse_band_part", "kmd_nccl_unique_id",
           "kmd_comm_init", "kmd_comm_destroy", "kmd_halo_exchange", "kmd_band_step",
           "kmd_host_workspace_bytes",
           "kmd_decode_filter_fuse_host", "kmd_decode_filter_fuse_host_bf16", "kmd_algorithmic_bytes", "kmd_launches_per_call",
           "kmd_status_string", "kmd_last_error", "kmd_version", "kmd_last_kernel")


def lib(build_if_missing: bool = True):
    """Load libkmd.so (building it in-tree first if it is missing or stale)."""
    global _lib
    if _lib is not None:
        return _lib
    if build_if_missing and LIB_PATH == _build.LIB and _build.is_stale():
        _build.build()
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libkmd.so not found at {LIB_PATH}; run __graft_entry__.build()")
    L = ctypes.CDLL(LIB_PATH)
    P, i32 = ctypes.c_void_p, ctypes.c_int32
    C = ctypes.POINTER(kmd_config)
    L.kmd_decode_filter_fuse.argtypes = [P, P, P, P, i32, i32, i32, C, P]
    L.kmd_decode_filter_fuse_remod.argtypes = [P, P, P, P, P, i32, i32, i32, C, P]
    L.kmd_decode_filter_fuse_bf16.argtypes = [P, P, P, P, i32, i32, i32, C, P]
    L.kmd_demodulate.argtypes = [P, P, ctypes.c_float, P, i32, i32, i32, P]
    L.kmd_remodulate.argtypes = [P, P, P, i32, i32, i32, P]
    L.kmd_decode_filter.argtypes = [P, P, P, i32, i32, i32, i32, P]
    MC = ctypes.POINTER(kmd_mr_config)
    L.kmd_mr_workspace_bytes.argtypes = [i32, i32, i32, MC]
    L.kmd_mr_workspace_bytes.restype = ctypes.c_size_t
    PP = ctypes.POINTER(ctypes.c_void_p)
    L.kmd_mr_decode_filter_fuse.argtypes = [P, PP, PP, PP, P, i32, i32, i32, MC, P, ctypes.c_size_t, P]
    L.kmd_downsample2x2.argtypes = [P, P, i32, i32, i32, i32, P]
    L.kmd_combine_resolutions.argtypes = [P, P, P, P, i32, i32, i32, P]
    L.kmd_fuse.argtypes = [P, P, P, i32, i32, i32, i32, i32, P]
    f32 = ctypes.c_float
    L.kmd_temporal_accumulate.argtypes = [P, P, P, P, P, P, P, P, P, P, i32, i32, i32, f32, f32, f32, P]
    L.kmd_backward_workspace_bytes.argtypes = [i32, i32, i32, C]
    L.kmd_backward_workspace_bytes.restype = ctypes.c_size_t
    L.kmd_decode_filter_fuse_backward.argtypes = [P, P, P, P, P, P, i32, i32, i32, C, P, ctypes.c_size_t, P]
    L.kmd_decode_filter_fuse_band.argtypes = [P, P, P, P, i32, i32, i32, i32, i32, i32, i32, C, P]
    L.kmd_decode_filter_fuse_band_part.argtypes = [P, P, P, P, i32, i32, i32, i32, i32, i32, i32, C, i32, P]
    L.kmd_nccl_unique_id.argtypes = [P]
    L.kmd_comm_init.argtypes = [PP, P, i32, i32]
    L.kmd_comm_destroy.argtypes = [P]
    L.kmd_halo_exchange.argtypes = [P, PP, i32, i32, i32, i32, i32, i32, P]
    L.kmd_band_step.argtypes = [P, P, P, P, P, i32, i32, i32, i32, i32, i32, i32, i32, C, P, P]
    L.kmd_host_workspace_bytes.argtypes = [i32, i32, i32, C]
    L.kmd_host_workspace_bytes.restype = ctypes.c_size_t
    L.kmd_decode_filter_fuse_host.argtypes = [P, P, P, P, i32, i32, i32, C, P, ctypes.c_size_t, P]
    L.kmd_decode_filter_fuse_host_bf16.argtypes = [P, P, P, P, i32, i32, i32, C, P, ctypes.c_size_t, P]
    L.kmd_algorithmic_bytes.argtypes = [i32, i32, i32, C, i32]
    L.kmd_algorithmic_bytes.restype = ctypes.c_int64
    L.kmd_launches_per_call.argtypes = []
    L.kmd_status_string.argtypes = [ctypes.c_int]
    L.kmd_status_string.restype = ctypes.c_char_p
    L.kmd_last_error.argtypes = []
    L.kmd_last_error.restype = ctypes.c_char_p
    L.kmd_version.argtypes = []
    L.kmd_last_kernel.argtypes = []
    L.kmd_last_kernel.restype = ctypes.c_int32
    for f in ("kmd_decode_filter_fuse", "kmd_decode_filter_fuse_bf16", "kmd_decode_filter_fuse_remod",
              "kmd_demodulate",
              "kmd_remodulate", "kmd_decode_filter", "kmd_fuse", "kmd_mr_decode_filter_fuse",
              "kmd_downsample2x2", "kmd_combine_resolutions", "kmd_decode_filter_fuse_backward",
              "kmd_temporal_accumulate",
              "kmd_decode_filter_fuse_band", "kmd_decode_filter_fuse_host",
              "kmd_decode_filter_fuse_band_part", "kmd_nccl_unique_id", "kmd_comm_init", "kmd_comm_destroy",
              "kmd_halo_exchange", "kmd_band_step"):
        getattr(L, f).restype = ctypes.c_int
    _lib = L
    return L


def _check(status: int):
    if status != 0:
        raise KmdError(status, lib().kmd_last_error().decode())


def _dev_f32(name: str, t: torch.Tensor, shape=None, dtype=torch.float32) -> int:
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {str(dtype).replace('torch.', '')}, got {t.dtype}")
    if t.device.type != "cuda":
        raise ValueError(f"{name} must be a CUDA tensor (libkmd has no CPU path)")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")
    return t.data_ptr()


def _on_one_device(fn):
    """Every tensor argument of a libkmd call must live on one CUDA device; the
    call runs with that device current (libkmd queries the current device for
    its SM count, function attributes and helper streams)."""
    import functools

    @functools.wraps(fn)
    def wrapped(*args, **kwargs):
        devs = set()

        def visit(v):
            if isinstance(v, torch.Tensor):
                if v.device.type == "cuda":
                    devs.add(v.device)
            elif isinstance(v, (list, tuple)):
                for u in v:
                    visit(u)
        for v in list(args) + list(kwargs.values()):
            visit(v)
        if len(devs) > 1:
            raise ValueError(f"{fn.__name__}: tensors on several devices {sorted(map(str, devs))}")
        if not devs:
            return fn(*args, **kwargs)
        with torch.cuda.device(devs.pop()):
            return fn(*args, **kwargs)
    return wrapped


def _stream(t: torch.Tensor, stream) -> int:
    if stream is None:
        stream = torch.cuda.current_stream(t.device)
    return stream.cuda_stream


@_on_one_device
def decode_filter_fuse(radiance: torch.Tensor, importance: torch.Tensor,
                       blend: Optional[torch.Tensor], sizes: Sequence[int],
                       out: Optional[torch.Tensor] = None, blend_is_logits: bool = True,
                       stream: Optional[torch.cuda.Stream] = None,
                       albedo: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Fused Eq. 3 -> 4 -> 5: radiance [N,3,H,W], importance [N,M,H,W],
    blend [N,M,H,W] (None iff M==1) -> out [N,3,H,W] (fp32, CUDA).  With
    ``albedo`` [N,3,H,W] the result is remodulated in the same pass
    (out = Rhat * albedo).  bfloat16 importance / blend
    (both, radiance stays fp32) select kmd_decode_filter_fuse_bf16 (W % 8 == 0)."""
    N, C, H, W = radiance.shape
    M = len(sizes)
    in16 = isinstance(importance, torch.Tensor) and importance.dtype == torch.bfloat16
    idt = torch.bfloat16 if in16 else torch.float32
    rp = _dev_f32("radiance", radiance, (N, 3, H, W))
    ip = _dev_f32("importance", importance, (N, M, H, W), idt)
    bp = None if blend is None else _dev_f32("blend", blend, (N, M, H, W), idt)
    if out is None:
        out = torch.empty((N, 3, H, W), device=radiance.device, dtype=torch.float32)
    op = _dev_f32("out", out, (N, 3, H, W))
    cfg = make_config(sizes, blend_is_logits)
    if in16:
        if albedo is not None:
            raise ValueError("albedo remodulation is not available with bf16 inputs")
        _check(lib().kmd_decode_filter_fuse_bf16(rp, ip, bp, op, N, H, W, ctypes.byref(cfg),
                                                 _stream(radiance, stream)))
    elif albedo is None:
        _check(lib().kmd_decode_filter_fuse(rp, ip, bp, op, N, H, W, ctypes.byref(cfg),
                                            _stream(radiance, stream)))
    else:
        ap = _dev_f32("albedo", albedo, (N, 3, H, W))
        _check(lib().kmd_decode_filter_fuse_remod(rp, ip, bp, ap, op, N, H, W, ctypes.byref(cfg),
                                                  _stream(radiance, stream)))
    return out


@_on_one_device
def demodulate(radiance: torch.Tensor, albedo: torch.Tensor, eps: float = 1e-3,
               out: Optional[torch.Tensor] = None,
               stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """irradiance = radiance / max(albedo, eps), [N,3,H,W] CUDA."""
    N, _, H, W = radiance.shape
    rp = _dev_f32("radiance", radiance, (N, 3, H, W))
    ap = _dev_f32("albedo", albedo, (N, 3, H, W))
    if out is None:
        out = torch.empty_like(radiance)
    op = _dev_f32("out", out, (N, 3, H, W))
    _check(lib().kmd_demodulate(rp, ap, float(eps), op, N, H, W, _stream(radiance, stream)))
    return out


@_on_one_device
def remodulate(irradiance: torch.Tensor, albedo: torch.Tensor, out: Optional[torch.Tensor] = None,
               stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """out = irradiance * albedo, [N,3,H,W] CUDA."""
    N, _, H, W = irradiance.shape
    xp = _dev_f32("irradiance", irradiance, (N, 3, H, W))
    ap = _dev_f32("albedo", albedo, (N, 3, H, W))
    if out is None:
        out = torch.empty_like(irradiance)
    op = _dev_f32("out", out, (N, 3, H, W))
    _check(lib().kmd_remodulate(xp, ap, op, N, H, W, _stream(irradiance, stream)))
    return out


@_on_one_device
def decode_filter(radiance: torch.Tensor, importance_i: torch.Tensor, k: int,
                  out: Optional[torch.Tensor] = None,
                  stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """One size, Eq. 3 -> 4: radiance [N,3,H,W], importance_i [N,1,H,W] -> [N,3,H,W]."""
    N, _, H, W = radiance.shape
    rp = _dev_f32("radiance", radiance, (N, 3, H, W))
    ip = _dev_f32("importance_i", importance_i, (N, 1, H, W))
    if out is None:
        out = torch.empty((N, 3, H, W), device=radiance.device, dtype=torch.float32)
    op = _dev_f32("out", out, (N, 3, H, W))
    _check(lib().kmd_decode_filter(rp, ip, op, N, H, W, int(k), _stream(radiance, stream)))
    return out


@_on_one_device
def fuse(filtered: torch.Tensor, blend: Optional[torch.Tensor], blend_is_logits: bool = True,
         out: Optional[torch.Tensor] = None,
         stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """Eq. 5 only: filtered [N,M,3,H,W], blend [N,M,H,W] -> [N,3,H,W]."""
    N, M, _, H, W = filtered.shape
    fp = _dev_f32("filtered", filtered, (N, M, 3, H, W))
    bp = None if blend is None else _dev_f32("blend", blend, (N, M, H, W))
    if out is None:
        out = torch.empty((N, 3, H, W), device=filtered.device, dtype=torch.float32)
    op = _dev_f32("out", out, (N, 3, H, W))
    _check(lib().kmd_fuse(fp, bp, op, N, H, W, M, int(bool(blend_is_logits)),
                          _stream(filtered, stream)))
    return out


@_on_one_device
def decode_filter_fuse_band(radiance: torch.Tensor, importance: torch.Tensor,
                            blend: Optional[torch.Tensor], sizes: Sequence[int], *,
                            y0: int, band_rows: int, halo_top: int, halo_bot: int,
                            H_global: int, out: Optional[torch.Tensor] = None,
                            blend_is_logits: bool = True,
                            stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """Row band [y0, y0+band_rows) of an H_global-row frame.  radiance /
    importance hold rows [y0-halo_top, y0+band_rows+halo_bot); blend and out
    hold the band rows only."""
    N, _, R, W = radiance.shape
    M = len(sizes)
    assert R == halo_top + band_rows + halo_bot, "radiance rows != halo_top+band_rows+halo_bot"
    rp = _dev_f32("radiance", radiance, (N, 3, R, W))
    ip = _dev_f32("importance", importance, (N, M, R, W))
    bp = None if blend is None else _dev_f32("blend", blend, (N, M, band_rows, W))
    if out is None:
        out = torch.empty((N, 3, band_rows, W), device=radiance.device, dtype=torch.float32)
    op = _dev_f32("out", out, (N, 3, band_rows, W))
    cfg = make_config(sizes, blend_is_logits)
    _check(lib().kmd_decode_filter_fuse_band(rp, ip, bp, op, N, band_rows, W, halo_top, halo_bot,
                                             y0, H_global, ctypes.byref(cfg),
                                             _stream(radiance, stream)))
    return out


BAND_ALL, BAND_INTERIOR, BAND_SEAMS = 0, 1, 2


@_on_one_device
def decode_filter_fuse_band_part(radiance: torch.Tensor, importance: torch.Tensor,
                                 blend: Optional[torch.Tensor], sizes: Sequence[int], part: int, *,
                                 y0: int, band_rows: int, halo_top: int, halo_bot: int, H_global: int,
                                 out: torch.Tensor, blend_is_logits: bool = True,
                                 stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """One part of a row band (BAND_INTERIOR: rows that read owned rows only;
    BAND_SEAMS: the rest; BAND_ALL: both) into ``out`` [N,3,band_rows,W]."""
    N, _, R, W = radiance.shape
    M = len(sizes)
    assert R == halo_top + band_rows + halo_bot, "radiance rows != halo_top+band_rows+halo_bot"
    rp = _dev_f32("radiance", radiance, (N, 3, R, W))
    ip = _dev_f32("importance", importance, (N, M, R, W))
    bp = None if blend is None else _dev_f32("blend", blend, (N, M, band_rows, W))
    op = _dev_f32("out", out, (N, 3, band_rows, W))
    cfg = make_config(sizes, blend_is_logits)
    _check(lib().kmd_decode_filter_fuse_band_part(rp, ip, bp, op, N, band_rows, W, halo_top, halo_bot,
                                                  y0, H_global, ctypes.byref(cfg), int(part),
                                                  _stream(radiance, stream)))
    return out


# ------------------------------------------- NCCL row-band exchange (configs[3])
def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0 creates it; broadcast it to every rank)."""
    buf = (ctypes.c_uint8 * 128)()
    _check(lib().kmd_nccl_unique_id(buf))
    return bytes(buf)


class Comm:
    """An NCCL communicator owned by libkmd's caller (kmd_comm_init / kmd_comm_destroy)."""

    def __init__(self, uid: bytes, nranks: int, rank: int):
        assert len(uid) == 128
        self.handle = ctypes.c_void_p()
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
        _check(lib().kmd_comm_init(ctypes.byref(self.handle), buf, nranks, rank))
        self.nranks, self.rank = nranks, rank

    def destroy(self):
        if self.handle:
            _check(lib().kmd_comm_destroy(self.handle))
            self.handle = ctypes.c_void_p()


@_on_one_device
def halo_exchange(comm: Comm, planes: Sequence[torch.Tensor], band_rows: int, halo: int,
                  peer_up: int, peer_down: int, stream: Optional[torch.cuda.Stream] = None) -> None:
    """kmd_halo_exchange over contiguous [halo_top + band_rows + halo_bot, W] CUDA planes."""
    if not planes:
        return
    W = planes[0].shape[-1]
    ptrs = (ctypes.c_void_p * len(planes))(*[_dev_f32(f"planes[{k}]", t) for k, t in enumerate(planes)])
    _check(lib().kmd_halo_exchange(comm.handle if comm else None, ptrs, len(planes), band_rows, W, halo,
                                   peer_up, peer_down, _stream(planes[0], stream)))


@_on_one_device
def band_step(comm: Optional[Comm], radiance: torch.Tensor, importance: torch.Tensor,
              blend: Optional[torch.Tensor], sizes: Sequence[int], out: torch.Tensor, *,
              y0: int, band_rows: int, halo: int, peer_up: int, peer_down: int, H_global: int,
              blend_is_logits: bool = True, stream: Optional[torch.cuda.Stream] = None,
              comm_stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """kmd_band_step: halo exchange on ``comm_stream`` overlapped with the band
    interior on ``stream``, then the seams.  radiance / importance hold
    [N, C, halo_top + band_rows + halo_bot, W] with halo_top = halo if
    peer_up >= 0 else 0 (likewise the bottom)."""
    N, _, R, W = radiance.shape
    M = len(sizes)
    top = halo if peer_up >= 0 else 0
    bot = halo if peer_down >= 0 else 0
    assert R == top + band_rows + bot, "radiance rows != halo_top + band_rows + halo_bot"
    rp = _dev_f32("radiance", radiance, (N, 3, R, W))
    ip = _dev_f32("importance", importance, (N, M, R, W))
    bp = None if blend is None else _dev_f32("blend", blend, (N, M, band_rows, W))
    op = _dev_f32("out", out, (N, 3, band_rows, W))
    cfg = make_config(sizes, blend_is_logits)
    cs = None if comm_stream is None else comm_stream.cuda_stream
    _check(lib().kmd_band_step(comm.handle if comm else None, rp, ip, bp, op, N, band_rows, W, halo,
                               peer_up, peer_down, y0, H_global, ctypes.byref(cfg),
                               _stream(radiance, stream), cs))
    return out


def host_workspace_bytes(N: int, H: int, W: int, sizes: Sequence[int]) -> int:
    cfg = make_config(sizes)
    return int(lib().kmd_host_workspace_bytes(N, H, W, ctypes.byref(cfg)))


@_on_one_device
def decode_filter_fuse_host(radiance: torch.Tensor, importance: torch.Tensor,
                            blend: Optional[torch.Tensor], sizes: Sequence[int],
                            out: torch.Tensor, workspace: torch.Tensor,
                            blend_is_logits: bool = True,
                            stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """End-to-end from host (ideally pinned) CPU tensors: H2D copies, fused
    kernel and D2H copy, all enqueued by libkmd on ``stream``.  ``workspace`` is
    a CUDA uint8 tensor of >= host_workspace_bytes(...) bytes.  Returns ``out``
    (caller synchronises ``stream`` before reading it).  importance / blend in
    bfloat16 (both) take kmd_decode_filter_fuse_host_bf16."""
    N, _, H, W = radiance.shape
    M = len(sizes)
    in16 = importance.dtype == torch.bfloat16
    idt = torch.bfloat16 if in16 else torch.float32
    for name, t, shape, dt in (("radiance", radiance, (N, 3, H, W), torch.float32),
                               ("importance", importance, (N, M, H, W), idt),
                               ("out", out, (N, 3, H, W), torch.float32)):
        if t.device.type != "cpu" or t.dtype != dt or not t.is_contiguous() or tuple(t.shape) != shape:
            raise ValueError(f"{name} must be a contiguous {dt} CPU tensor of shape {shape}")
    if blend is not None and (blend.device.type != "cpu" or tuple(blend.shape) != (N, M, H, W)
                              or blend.dtype != idt or not blend.is_contiguous()):
        raise ValueError(f"blend must be a contiguous {idt} CPU tensor [N,M,H,W] (importance's dtype)")
    if workspace.device.type != "cuda":
        raise ValueError("workspace must be a CUDA tensor")
    cfg = make_config(sizes, blend_is_logits)
    if stream is None:
        stream = torch.cuda.current_stream(workspace.device)
    entry = lib().kmd_decode_filter_fuse_host_bf16 if in16 else lib().kmd_decode_filter_fuse_host
    _check(entry(
        radiance.data_ptr(), importance.data_ptr(),
        None if blend is None else blend.data_ptr(), out.data_ptr(), N, H, W,
        ctypes.byref(cfg), workspace.data_ptr(), workspace.numel() * workspace.element_size(),
        stream.cuda_stream))
    return out


def algorithmic_bytes(N: int, H: int, W: int, sizes: Sequence[int], has_blend: bool) -> int:
    cfg = make_config(sizes)
    return int(lib().kmd_algorithmic_bytes(N, H, W, ctypes.byref(cfg), int(bool(has_blend))))


def launches_per_call() -> int:
    return int(lib().kmd_launches_per_call())


LAST_KERNEL = {0: "none", 1: "v1-direct", 2: "v2-ws", 3: "v3-tma", 10: "bwd-tile", 11: "bwd-tma"}


def last_kernel() -> str:
    """Kernel variant of the last fused launch on this thread (diagnostic):
    v1-direct, v2-ws, v3-tma (runtime M), v3-tma-M<m>[-albedo] (compiled for M),
    v3-tma-bf16[-M<m>] (bf16 importance / logits)."""
    code = int(lib().kmd_last_kernel())
    if code >= 300:  # the multi-resolution levels' 28-row-tile kernel (+ Eq. 7 combine epilogue)
        return "v3-tma28-mr-cmb" if code == 301 else "v3-tma28-mr"
    if code >= 200:
        return f"v3-tma-bf16-M{code - 200}" if code > 200 else "v3-tma-bf16"
    if code >= 150:
        return f"v3-tma-M{code - 150}-albedo"
    if code >= 100:
        return f"v3-tma-M{code - 100}"
    return LAST_KERNEL.get(code, "?")


def version() -> int:
    return int(lib().kmd_version())


# --------------------------------------------- multi-resolution (NEXT row 2)
def mr_workspace_bytes(N: int, H: int, W: int, sizes_per_level) -> int:
    cfg = make_mr_config(sizes_per_level)
    return int(lib().kmd_mr_workspace_bytes(N, H, W, ctypes.byref(cfg)))


@_on_one_device
def mr_decode_filter_fuse(radiance: torch.Tensor, importance, blend, alpha, sizes_per_level,
                          out: Optional[torch.Tensor] = None,
                          workspace: Optional[torch.Tensor] = None,
                          stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """"Ours MR" (Eq. 7): radiance [N,3,H,W]; importance[l],
    blend[l] [N,M_l,H>>l,W>>l]; alpha[l] [N,1,H>>l,W>>l] for l < levels-1."""
    N, _, H, W = radiance.shape
    L = len(sizes_per_level)
    rp = _dev_f32("radiance", radiance, (N, 3, H, W))
    ip = (ctypes.c_void_p * L)(*[_dev_f32(f"importance[{l}]", importance[l],
                                         (N, len(sizes_per_level[l]), H >> l, W >> l))
                                 for l in range(L)])
    bp = None
    if blend is not None:
        bp = (ctypes.c_void_p * L)(*[None if blend[l] is None else
                                     _dev_f32(f"blend[{l}]", blend[l],
                                              (N, len(sizes_per_level[l]), H >> l, W >> l))
                                     for l in range(L)])
    ap = (ctypes.c_void_p * max(1, L - 1))(*[_dev_f32(f"alpha[{l}]", alpha[l], (N, 1, H >> l, W >> l))
                                             for l in range(L - 1)])
    if out is None:
        out = torch.empty((N, 3, H, W), device=radiance.device, dtype=torch.float32)
    op = _dev_f32("out", out, (N, 3, H, W))
    cfg = make_mr_config(sizes_per_level)
    need = int(lib().kmd_mr_workspace_bytes(N, H, W, ctypes.byref(cfg)))
    if workspace is None:
        workspace = torch.empty(need, dtype=torch.uint8, device=radiance.device)
    _check(lib().kmd_mr_decode_filter_fuse(
        rp, ctypes.cast(ip, ctypes.POINTER(ctypes.c_void_p)),
        None if bp is None else ctypes.cast(bp, ctypes.POINTER(ctypes.c_void_p)),
        ctypes.cast(ap, ctypes.POINTER(ctypes.c_void_p)), op, N, H, W, ctypes.byref(cfg),
        workspace.data_ptr(), workspace.numel(), _stream(radiance, stream)))
    return out


@_on_one_device
def downsample2x2(x: torch.Tensor, out: Optional[torch.Tensor] = None,
                  stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    N, C, H, W = x.shape
    xp = _dev_f32("in", x)
    if out is None:
        out = torch.empty((N, C, H // 2, W // 2), device=x.device, dtype=torch.float32)
    op = _dev_f32("out", out, (N, C, H // 2, W // 2))
    _check(lib().kmd_downsample2x2(xp, op, N, C, H, W, _stream(x, stream)))
    return out


@_on_one_device
def combine_resolutions(fine: torch.Tensor, coarse: torch.Tensor, alpha: torch.Tensor,
                        out: Optional[torch.Tensor] = None,
                        stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    N, _, H, W = fine.shape
    fp = _dev_f32("fine", fine, (N, 3, H, W))
    cp = _dev_f32("coarse", coarse, (N, 3, H // 2, W // 2))
    ap = _dev_f32("alpha", alpha, (N, 1, H, W))
    if out is None:
        out = torch.empty_like(fine)
    op = _dev_f32("out", out, (N, 3, H, W))
    _check(lib().kmd_combine_resolutions(fp, cp, ap, op, N, H, W, _stream(fine, stream)))
    return out


# ------------------------------------------------------- backward (NEXT row 3)
def backward_workspace_bytes(N: int, H: int, W: int, sizes: Sequence[int]) -> int:
    cfg = make_config(sizes)
    return int(lib().kmd_backward_workspace_bytes(N, H, W, ctypes.byref(cfg)))


@_on_one_device
def decode_filter_fuse_backward(radiance: torch.Tensor, importance: torch.Tensor,
                                blend: Optional[torch.Tensor], grad_out: torch.Tensor,
                                sizes: Sequence[int], blend_is_logits: bool = True,
                                grad_importance: Optional[torch.Tensor] = None,
                                grad_blend: Optional[torch.Tensor] = None,
                                workspace: Optional[torch.Tensor] = None,
                                stream: Optional[torch.cuda.Stream] = None):
    """dL/dI [N,M,H,W] and dL/dB [N,M,H,W] (None when blend is None) given
    grad_out = dL/dRhat [N,3,H,W] (Eq. 1: the decoder is
    trained end to end through Eq. 3-5)."""
    N, _, H, W = radiance.shape
    M = len(sizes)
    rp = _dev_f32("radiance", radiance, (N, 3, H, W))
    ip = _dev_f32("importance", importance, (N, M, H, W))
    bp = None if blend is None else _dev_f32("blend", blend, (N, M, H, W))
    gp = _dev_f32("grad_out", grad_out, (N, 3, H, W))
    if grad_importance is None:
        grad_importance = torch.empty((N, M, H, W), device=radiance.device, dtype=torch.float32)
    gip = _dev_f32("grad_importance", grad_importance, (N, M, H, W))
    gbp = None
    if blend is not None:
        if grad_blend is None:
            grad_blend = torch.empty((N, M, H, W), device=radiance.device, dtype=torch.float32)
        gbp = _dev_f32("grad_blend", grad_blend, (N, M, H, W))
    cfg = make_config(sizes, blend_is_logits)
    need = int(lib().kmd_backward_workspace_bytes(N, H, W, ctypes.byref(cfg)))
    if workspace is None:
        workspace = torch.empty(max(need, 1), dtype=torch.uint8, device=radiance.device)
    _check(lib().kmd_decode_filter_fuse_backward(rp, ip, bp, gp, gip, gbp, N, H, W, ctypes.byref(cfg),
                                                 workspace.data_ptr(), workspace.numel(),
                                                 _stream(radiance, stream)))
    return grad_importance, grad_blend


def backward_launches_per_call(M: int, path: Optional[str] = None, blend_is_logits: bool = True) -> int:
    """Kernel launches of one decode_filter_fuse_backward call: the TMA path
    ("bwd-tma") runs the log-sum-exp pass (M > 1 with logits), pass A, pass B
    and pass C (or a memset when M == 1); the one-launch tiled fallback
    ("bwd-tile") adds a memset when M == 1."""
    path = path or last_kernel()
    if path == "bwd-tma":
        return 4 if M > 1 and blend_is_logits else 3
    return 1 if M > 1 else 2


class DecodeFilterFuse(torch.autograd.Function):
    """Differentiable kmd_decode_filter_fuse (w.r.t. importance and blend):
    forward and backward both run in libkmd.  The backward evaluates exp(I)
    unshifted (include/kmd.h: importance in (-80, 80)); with ``check_range``
    (default) an importance map outside that range raises ValueError instead
    of returning inf / NaN gradients (one device reduction and one host sync
    per backward call)."""

    check_range = True
    IMPORTANCE_LIMIT = 80.0

    @staticmethod
    def forward(ctx, radiance, importance, blend, sizes, blend_is_logits=True):
        ctx.sizes = tuple(sizes)
        ctx.logits = blend_is_logits
        ctx.save_for_backward(radiance, importance, blend)
        return decode_filter_fuse(radiance, importance, blend, sizes, blend_is_logits=blend_is_logits)

    @staticmethod
    def backward(ctx, grad_out):
        radiance, importance, blend = ctx.saved_tensors
        if DecodeFilterFuse.check_range and importance.numel() > 0:
            m = float(importance.abs().amax())
            if not m < DecodeFilterFuse.IMPORTANCE_LIMIT:
                raise ValueError(f"DecodeFilterFuse.backward: max |importance| = {m:g} is outside the "
                                 f"backward's range (-{DecodeFilterFuse.IMPORTANCE_LIMIT:g}, "
                                 f"{DecodeFilterFuse.IMPORTANCE_LIMIT:g}) (include/kmd.h); "
                                 "shift the importance maps (the decoder is shift-invariant, PAPER.md:154)")
        gI, gB = decode_filter_fuse_backward(radiance, importance, blend, grad_out.contiguous(),
                                             ctx.sizes, ctx.logits)
        return None, gI, gB, None, None


# ------------------------------------------------ temporal accumulation (NEXT row 4)
@_on_one_device
def temporal_accumulate(cur_rad: torch.Tensor, prev_rad: torch.Tensor, prev_pos: torch.Tensor,
                        prev_nrm: torch.Tensor, prev_valid: torch.Tensor, cur_pos: torch.Tensor,
                        cur_nrm: torch.Tensor, motion: torch.Tensor, pos_tol: float,
                        normal_tol: float = 0.9, alpha: float = 0.2,
                        accum: Optional[torch.Tensor] = None, mask: Optional[torch.Tensor] = None,
                        want_mask: bool = True, stream: Optional[torch.cuda.Stream] = None):
    """Reproject + consistency test + accumulate (§4.1)
    in one kernel: returns (accum [N,3,H,W] fp32, mask [N,H,W] uint8 or None)."""
    N, _, H, W = cur_rad.shape
    ptrs = [_dev_f32(nm, t, (N, 3, H, W)) for nm, t in (("cur_rad", cur_rad), ("prev_rad", prev_rad),
                                                        ("prev_pos", prev_pos), ("prev_nrm", prev_nrm))]
    if prev_valid.dtype != torch.uint8 or prev_valid.device.type != "cuda" or not prev_valid.is_contiguous() \
            or tuple(prev_valid.shape) != (N, H, W):
        raise ValueError("prev_valid must be a contiguous CUDA uint8 tensor [N,H,W]")
    cp = _dev_f32("cur_pos", cur_pos, (N, 3, H, W))
    cn = _dev_f32("cur_nrm", cur_nrm, (N, 3, H, W))
    mo = _dev_f32("motion", motion, (N, 2, H, W))
    if accum is None:
        accum = torch.empty((N, 3, H, W), device=cur_rad.device, dtype=torch.float32)
    ap = _dev_f32("accum", accum, (N, 3, H, W))
    mp = None
    if want_mask:
        if mask is None:
            mask = torch.empty((N, H, W), device=cur_rad.device, dtype=torch.uint8)
        if mask.dtype != torch.uint8 or tuple(mask.shape) != (N, H, W) or not mask.is_contiguous():
            raise ValueError("mask must be a contiguous uint8 tensor [N,H,W]")
        mp = mask.data_ptr()
    _check(lib().kmd_temporal_accumulate(*ptrs, prev_valid.data_ptr(), cp, cn, mo, ap, mp, N, H, W,
                                         float(pos_tol), float(normal_tol), float(alpha),
                                         _stream(cur_rad, stream)))
    return accum, (mask if want_mask else None)
