"""CPU oracle for the kernel-map decoder + filter + fusion (arXiv 2202.05977).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_2202_05977_b200``) never imports it, and
nothing here imports the product package: the two share no code.

The arithmetic lives in ``kmd_oracle.c`` (plain C, fp64, literal Eq. 3 -> 4
-> 5 of PAPER.md, see the citations there).  This module only builds that
library with gcc and marshals numpy arrays to it.

Every function is pinned by ``tests/test_oracle_pins.py``; none is
"parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "kmd_oracle.c")
_HDR = os.path.join(_HERE, "kmd_oracle.h")
LIB_PATH = os.path.join(_HERE, "libkmd_oracle.so")

_lib = None

_ERRORS = {1: "NULL pointer", 2: "bad config (size/M)", 3: "bad dimension/index", 4: "out of memory"}


class OracleError(RuntimeError):
    pass


def build(force: bool = False) -> str:
    """Compile kmd_oracle.c with gcc (-O2, OpenMP, strict IEEE: no -ffast-math)."""
    stale = (not os.path.exists(LIB_PATH)) or any(
        os.path.getmtime(p) > os.path.getmtime(LIB_PATH) for p in (_SRC, _HDR))
    if force or stale:
        tmp = LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-ffp-contract=off", "-Wall", "-Wextra", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, LIB_PATH)
    return LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(LIB_PATH)
        P = ctypes.c_void_p
        i32 = ctypes.c_int32
        lib.kmdo_unfold.argtypes = [P, i32, i32, i32, P]
        lib.kmdo_kernel_map.argtypes = [P, i32, i32, i32, P]
        lib.kmdo_apply.argtypes = [P, i32, P, i32, i32, P]
        lib.kmdo_fuse.argtypes = [P, P, i32, i32, i32, i32, P]
        lib.kmdo_decode_filter_fuse_rows.argtypes = [P, P, P, i32, i32, i32, i32, P, i32,
                                                     i32, i32, i32, P]
        lib.kmdo_decode_filter_fuse_rows_f64rad.argtypes = [P, P, P, i32, i32, i32, i32, P, i32,
                                                            i32, i32, i32, P]
        lib.kmdo_decode_filter_fuse_pixels.argtypes = [P, P, P, i32, i32, i32, i32, P, i32,
                                                       P, P, P, ctypes.c_int64, i32, P]
        lib.kmdo_max_threads.argtypes = []
        lib.kmdo_demodulate.argtypes = [P, P, ctypes.c_double, ctypes.c_int64, P]
        lib.kmdo_remodulate.argtypes = [P, P, ctypes.c_int64, P]
        lib.kmdo_downsample_2x2.argtypes = [P, ctypes.c_int64, i32, i32, P]
        lib.kmdo_upsample_nearest.argtypes = [P, ctypes.c_int64, i32, i32, P]
        lib.kmdo_combine_resolutions.argtypes = [P, P, P, i32, i32, i32, P]
        lib.kmdo_backward.argtypes = [P, P, P, P, i32, i32, i32, i32, P, i32, P, P]
        f32 = ctypes.c_float
        lib.kmdo_temporal_accumulate.argtypes = [P, P, P, P, P, P, P, P, i32, i32, i32, f32, f32, f32, P, P]
        for f in ("kmdo_unfold", "kmdo_kernel_map", "kmdo_apply", "kmdo_fuse",
                  "kmdo_decode_filter_fuse_rows", "kmdo_decode_filter_fuse_rows_f64rad",
                  "kmdo_decode_filter_fuse_pixels",
                  "kmdo_max_threads", "kmdo_demodulate", "kmdo_remodulate", "kmdo_downsample_2x2",
                  "kmdo_upsample_nearest", "kmdo_combine_resolutions", "kmdo_backward",
                  "kmdo_temporal_accumulate"):
            getattr(lib, f).restype = ctypes.c_int
        _lib = lib
    return _lib


def _check(st: int):
    if st != 0:
        raise OracleError(f"oracle error {st}: {_ERRORS.get(st, '?')}")


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32))


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def max_threads() -> int:
    return int(_load().kmdo_max_threads())


# ---------------------------------------------------------------- explicit path
def unfold(imap, k: int) -> np.ndarray:
    """Fig. 3 unfold of an [H,W] map -> [H,W,k*k] (fp64), clamp-to-edge."""
    imap = _f32(imap)
    H, W = imap.shape
    out = np.empty((H, W, k * k), dtype=np.float64)
    _check(_load().kmdo_unfold(_ptr(imap), H, W, k, _ptr(out)))
    return out


def kernel_map(imap, k: int) -> np.ndarray:
    """Eq. 3: the explicit H x W x k^2 kernel map (softmax along channels)."""
    imap = _f32(imap)
    H, W = imap.shape
    out = np.empty((H, W, k * k), dtype=np.float64)
    _check(_load().kmdo_kernel_map(_ptr(imap), H, W, k, _ptr(out)))
    return out


def apply(kmap: np.ndarray, k: int, radiance) -> np.ndarray:
    """Eq. 4: apply an explicit kernel map to radiance [3,H,W] -> [3,H,W] fp64."""
    radiance = _f32(radiance)
    kmap = np.ascontiguousarray(kmap, dtype=np.float64)
    _, H, W = radiance.shape
    assert kmap.shape == (H, W, k * k)
    out = np.empty((3, H, W), dtype=np.float64)
    _check(_load().kmdo_apply(_ptr(kmap), k, _ptr(radiance), H, W, _ptr(out)))
    return out


def fuse(filtered: np.ndarray, blend, blend_is_logits: bool = True) -> np.ndarray:
    """Eq. 5: filtered [M,3,H,W] (fp64), blend [M,H,W] (or None iff M==1) -> [3,H,W]."""
    filtered = np.ascontiguousarray(filtered, dtype=np.float64)
    M, _, H, W = filtered.shape
    b = None if blend is None else _f32(blend)
    out = np.empty((3, H, W), dtype=np.float64)
    _check(_load().kmdo_fuse(_ptr(filtered), _ptr(b), M, H, W, int(bool(blend_is_logits)),
                             _ptr(out)))
    return out


def explicit_decode_filter_fuse(radiance, importance, blend, sizes: Sequence[int],
                                blend_is_logits: bool = True) -> np.ndarray:
    """KPCN-style composition for ONE frame: materialise every kernel map
    (unfold -> Eq. 3), apply it (Eq. 4), then fuse (Eq. 5).  Small inputs only."""
    radiance = _f32(radiance)
    importance = _f32(importance)
    M = len(sizes)
    filtered = np.stack([apply(kernel_map(importance[i], k), k, radiance)
                         for i, k in enumerate(sizes)])
    return fuse(filtered, blend if M > 1 else None, blend_is_logits)


# --------------------------------------------------------------- streaming path
def decode_filter_fuse(radiance, importance, blend, sizes: Sequence[int],
                       blend_is_logits: bool = True, rows: Optional[tuple] = None,
                       threads: int = 0) -> np.ndarray:
    """Per-pixel evaluation of Eq. 3 -> 4 -> 5 for radiance [N,3,H,W],
    importance [N,M,H,W], blend [N,M,H,W] (None iff M==1).  Returns fp64
    [N,3,H,W], or [N,3,y1-y0,W] for rows=(y0,y1)."""
    f64 = isinstance(radiance, np.ndarray) and radiance.dtype == np.float64
    radiance = np.ascontiguousarray(radiance) if f64 else _f32(radiance)
    importance = _f32(importance)
    b = None if blend is None else _f32(blend)
    N, _, H, W = radiance.shape
    M = importance.shape[1]
    assert len(sizes) == M
    y0, y1 = (0, H) if rows is None else rows
    sz = np.ascontiguousarray(sizes, dtype=np.int32)
    out = np.empty((N, 3, y1 - y0, W), dtype=np.float64)
    # fp64 radiance (the multi-resolution pyramid levels) is read as given
    fn = _load().kmdo_decode_filter_fuse_rows_f64rad if f64 else _load().kmdo_decode_filter_fuse_rows
    _check(fn(_ptr(radiance), _ptr(importance), _ptr(b), N, H, W, M, _ptr(sz),
              int(bool(blend_is_logits)), y0, y1, threads, _ptr(out)))
    return out


def decode_filter_fuse_pixels(radiance, importance, blend, sizes: Sequence[int],
                              n, y, x, blend_is_logits: bool = True,
                              threads: int = 0) -> np.ndarray:
    """Per-pixel evaluation at the listed (n, y, x) positions -> [count, 3] fp64."""
    radiance = _f32(radiance)
    importance = _f32(importance)
    b = None if blend is None else _f32(blend)
    N, _, H, W = radiance.shape
    M = importance.shape[1]
    assert len(sizes) == M
    n = np.ascontiguousarray(n, dtype=np.int32)
    y = np.ascontiguousarray(y, dtype=np.int32)
    x = np.ascontiguousarray(x, dtype=np.int32)
    sz = np.ascontiguousarray(sizes, dtype=np.int32)
    out = np.empty((len(n), 3), dtype=np.float64)
    _check(_load().kmdo_decode_filter_fuse_pixels(
        _ptr(radiance), _ptr(importance), _ptr(b), N, H, W, M, _ptr(sz),
        int(bool(blend_is_logits)), _ptr(n), _ptr(y), _ptr(x), len(n), threads, _ptr(out)))
    return out


# ------------------------------------------------------ albedo (NEXT row 1)
def demodulate(radiance, albedo, eps: float = 1e-3) -> np.ndarray:
    """irradiance = radiance / max(albedo, eps) (fp64)."""
    r = _f32(radiance)
    a = _f32(albedo)
    assert r.shape == a.shape
    out = np.empty(r.shape, dtype=np.float64)
    _check(_load().kmdo_demodulate(_ptr(r), _ptr(a), float(eps), r.size, _ptr(out)))
    return out


def remodulate(irradiance, albedo) -> np.ndarray:
    """SPEC.md:138-145 / PAPER.md:181: out = irradiance * albedo (fp64)."""
    x = np.ascontiguousarray(irradiance, dtype=np.float64)
    a = _f32(albedo)
    assert x.shape == a.shape
    out = np.empty(x.shape, dtype=np.float64)
    _check(_load().kmdo_remodulate(_ptr(x), _ptr(a), x.size, _ptr(out)))
    return out


# ---------------------------------- multi-resolution "Ours MR" (NEXT row 2)
def downsample_2x2(img) -> np.ndarray:
    """D of Eq. 7: [..., H, W] fp32 -> [..., H/2, W/2] fp64 block means."""
    a = _f32(img)
    H, W = a.shape[-2:]
    out = np.empty(a.shape[:-2] + (H // 2, W // 2), dtype=np.float64)
    _check(_load().kmdo_downsample_2x2(_ptr(a), a.size // (H * W), H, W, _ptr(out)))
    return out


def downsample_2x2_f64(img) -> np.ndarray:
    """D of Eq. 7 on an fp32 or fp64 image, in fp64: the block mean written out
    (SPEC.md:56-63), for the pyramid's deeper levels."""
    a = np.asarray(img, dtype=np.float64)
    return 0.25 * ((a[..., 0::2, 0::2] + a[..., 0::2, 1::2]) + (a[..., 1::2, 0::2] + a[..., 1::2, 1::2]))


def upsample_nearest(img) -> np.ndarray:
    """U of Eq. 7: [..., h, w] -> [..., 2h, 2w] (fp64)."""
    a = np.ascontiguousarray(img, dtype=np.float64)
    h, w = a.shape[-2:]
    out = np.empty(a.shape[:-2] + (2 * h, 2 * w), dtype=np.float64)
    _check(_load().kmdo_upsample_nearest(_ptr(a), a.size // (h * w), h, w, _ptr(out)))
    return out


def combine_resolutions(fine, coarse, alpha) -> np.ndarray:
    """Eq. 7: fine [N,3,H,W], coarse [N,3,H/2,W/2], alpha [N,1,H,W]."""
    f = np.ascontiguousarray(fine, dtype=np.float64)
    c = np.ascontiguousarray(coarse, dtype=np.float64)
    a = _f32(alpha)
    N, _, H, W = f.shape
    out = np.empty_like(f)
    _check(_load().kmdo_combine_resolutions(_ptr(f), _ptr(c), _ptr(a), N, H, W, _ptr(out)))
    return out


def mr_decode_filter_fuse(radiance, importance, blend, alpha, sizes, threads: int = 0) -> np.ndarray:
    """"Ours MR": level l filters D^l(radiance) with importance[l], blend[l]
    (Eq. 3-5), then Eq. 7 combines from the coarsest level.  The pyramid
    levels D^l(radiance) stay in fp64 (PAPER.md:316-318 defines them exactly)."""
    L = len(importance)
    rad = [_f32(radiance)]
    for _ in range(1, L):
        rad.append(downsample_2x2_f64(rad[-1]))
    f = [decode_filter_fuse(rad[l], importance[l], None if blend is None else blend[l], sizes[l],
                            threads=threads) for l in range(L)]
    c = f[L - 1]
    for l in range(L - 2, -1, -1):
        c = combine_resolutions(f[l], c, alpha[l])
    return c


# ------------------------------------------------------- backward (NEXT row 3)
def backward(radiance, importance, blend, grad_out, sizes, blend_is_logits: bool = True):
    """dL/dI [N,M,H,W] and dL/dB [N,M,H,W] (fp64) for L with dL/dRhat = grad_out."""
    radiance = _f32(radiance)
    importance = _f32(importance)
    b = None if blend is None else _f32(blend)
    G = np.ascontiguousarray(grad_out, dtype=np.float64)
    N, _, H, W = radiance.shape
    M = importance.shape[1]
    sz = np.ascontiguousarray(sizes, dtype=np.int32)
    gI = np.empty((N, M, H, W), dtype=np.float64)
    gB = np.empty((N, M, H, W), dtype=np.float64)
    _check(_load().kmdo_backward(_ptr(radiance), _ptr(importance), _ptr(b), _ptr(G), N, H, W, M,
                                 _ptr(sz), int(bool(blend_is_logits)), _ptr(gI), _ptr(gB)))
    return gI, gB


# ------------------------------------------------ temporal accumulation (NEXT row 4)
def temporal_accumulate(cur_rad, prev_rad, prev_pos, prev_nrm, prev_valid, cur_pos, cur_nrm, motion,
                        pos_tol: float, normal_tol: float = 0.9, alpha: float = 0.2):
    """reproject + consistency_test + temporal_accumulate:
    returns (accum [N,3,H,W] fp64, mask [N,H,W] uint8)."""
    arrs = [_f32(a) for a in (cur_rad, prev_rad, prev_pos, prev_nrm)]
    valid = np.ascontiguousarray(prev_valid, dtype=np.uint8)
    cp, cn, mo = _f32(cur_pos), _f32(cur_nrm), _f32(motion)
    N, _, H, W = arrs[0].shape
    accum = np.empty((N, 3, H, W), dtype=np.float64)
    mask = np.empty((N, H, W), dtype=np.uint8)
    _check(_load().kmdo_temporal_accumulate(*[_ptr(a) for a in arrs], _ptr(valid), _ptr(cp), _ptr(cn),
                                            _ptr(mo), N, H, W, float(pos_tol), float(normal_tol),
                                            float(alpha), _ptr(accum), _ptr(mask)))
    return accum, mask
