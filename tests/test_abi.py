"""C-ABI contract of libkmd that needs no GPU: the library loads, exports every
function include/kmd.h declares, and rejects bad arguments with the documented
status codes before touching CUDA (argument checks run first, kmd.h)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2202_05977_b200 import kmd
    return kmd.lib()


@pytest.fixture(scope="module")
def kmdmod():
    from paper_2202_05977_b200 import kmd
    return kmd


def _declared_functions():
    src = open(os.path.join(ROOT, "include", "kmd.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(kmd_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = _declared_functions()
    for must in ("kmd_decode_filter_fuse", "kmd_decode_filter", "kmd_fuse",
                 "kmd_decode_filter_fuse_band", "kmd_decode_filter_fuse_host"):
        assert must in names


def test_library_exports_every_declared_symbol(L):
    for name in _declared_functions():
        assert hasattr(L, name), f"libkmd.so does not export {name}"


def test_status_strings_and_version(L):
    for code, name in [(0, b"KMD_OK"), (2, b"KMD_ERR_CONFIG"), (5, b"KMD_ERR_ALIAS"),
                       (6, b"KMD_ERR_CUDA")]:
        assert L.kmd_status_string(code) == name
    assert L.kmd_version() == 1
    assert L.kmd_launches_per_call() >= 1


def _call(L, kmdmod, sizes, N=1, H=64, W=64, rad=0x1000, imp=0x100000, blend=0x200000,
          out=0x40000000, logits=1):
    cfg = kmdmod.make_config(sizes)
    cfg.blend_is_logits = logits
    return L.kmd_decode_filter_fuse(rad, imp, blend, out, N, H, W, ctypes.byref(cfg), None)


def test_config_errors(L, kmdmod):
    assert _call(L, kmdmod, [3, 4]) == 2                 # even k
    assert _call(L, kmdmod, [0]) == 2                    # k < 1
    assert _call(L, kmdmod, [33]) == 2                   # k > KMD_MAX_K
    assert _call(L, kmdmod, [13], H=12) == 2             # k > min(H, W)
    assert _call(L, kmdmod, [3] * 9) == 2                # M > 8
    assert _call(L, kmdmod, []) == 2                     # M < 1
    assert _call(L, kmdmod, [3], logits=2) == 2
    assert _call(L, kmdmod, [3, 4]) == 2
    assert b"sizes[1]" in L.kmd_last_error()


def test_null_dim_alias_errors(L, kmdmod):
    assert _call(L, kmdmod, [3, 5], blend=None) == 1     # M > 1 needs blend
    assert _call(L, kmdmod, [3], rad=None) == 1
    assert _call(L, kmdmod, [3], N=-1) == 3
    assert _call(L, kmdmod, [3], W=0) == 3
    assert _call(L, kmdmod, [3], out=0x1000 + 64) == 5   # out overlaps radiance
    assert _call(L, kmdmod, [3, 5], out=0x200000 + 4) == 5  # out overlaps blend
    cfg = kmdmod.make_config([3])
    # N == 0 is a no-op (empty tensors have NULL data pointers)
    assert L.kmd_decode_filter_fuse(None, None, None, None, 0, 0, 0, ctypes.byref(cfg), None) == 0
    assert L.kmd_decode_filter_fuse(None, 0x20, None, 0x30, 1, 8, 8, ctypes.byref(cfg), None) == 1


def test_band_geometry_errors(L, kmdmod):
    cfg = kmdmod.make_config([3, 13])
    f = L.kmd_decode_filter_fuse_band
    args = (0x1000, 0x1000000, 0x2000000, 0x40000000)
    # halo smaller than r_max = 6 at an interior band
    assert f(*args, 1, 100, 64, 5, 6, 100, 400, ctypes.byref(cfg), None) == 3
    # band beyond the frame
    assert f(*args, 1, 100, 64, 6, 6, 300, 400, ctypes.byref(cfg), None) == 3
    # bottom halo 5 < r_max = 6 for a band that does not reach the frame bottom
    assert f(*args, 1, 100, 64, 0, 5, 0, 400, ctypes.byref(cfg), None) == 3


def test_fuse_errors(L):
    assert L.kmd_fuse(0x1000, None, 0x100000, 1, 8, 8, 2, 1, None) == 1
    assert L.kmd_fuse(0x1000, 0x2000, 0x100000, 1, 8, 8, 9, 1, None) == 2
    assert L.kmd_fuse(0x1000, 0x2000, 0x1000, 1, 8, 8, 2, 1, None) == 5


def test_algorithmic_bytes(kmdmod):
    # 72 B/px at M=6 with blend; 28 B/px at M=1 without
    assert kmdmod.algorithmic_bytes(1, 1080, 1920, [3, 5, 7, 9, 11, 13], True) == 72 * 1920 * 1080
    assert kmdmod.algorithmic_bytes(1, 64, 64, [5], False) == 28 * 64 * 64


def test_binding_rejects_cpu_tensors(kmdmod):
    import torch
    x = torch.zeros(1, 3, 8, 8)
    with pytest.raises(ValueError, match="CUDA"):
        kmdmod.decode_filter_fuse(x, torch.zeros(1, 1, 8, 8), None, [3])


def test_bf16_entry_point_errors(L, kmdmod):
    # kmd_decode_filter_fuse_bf16 (NEXT row 4's alternative): checks precede CUDA
    f = L.kmd_decode_filter_fuse_bf16
    cfg = kmdmod.make_config([3, 5])
    args = (0x1000, 0x100000, 0x200000, 0x40000000)
    assert f(*args, 1, 64, 60, ctypes.byref(cfg), None) == 4          # W % 8 != 0
    assert f(0x1004, *args[1:], 1, 64, 64, ctypes.byref(cfg), None) == 4  # misaligned radiance
    assert f(*args[:2], None, args[3], 1, 64, 64, ctypes.byref(cfg), None) == 1  # M > 1 needs blend
    assert f(*args[:3], 0x100000 + 16, 1, 64, 64, ctypes.byref(cfg), None) == 5  # out overlaps importance
    assert f(*args, 1, 64, 64, ctypes.byref(kmdmod.make_config([3, 15])), None) == 2  # k > 13
    assert f(*args, -1, 64, 64, ctypes.byref(cfg), None) == 3
    assert f(None, None, None, None, 0, 0, 0, ctypes.byref(cfg), None) == 0  # N == 0: no-op


def test_binding_bf16_dtype_checks(kmdmod):
    import torch
    x = torch.zeros(1, 3, 8, 8)
    with pytest.raises(ValueError, match="CUDA"):
        kmdmod.decode_filter_fuse(x, torch.zeros(1, 1, 8, 8, dtype=torch.bfloat16), None, [3])


def test_backward_workspace_formula(kmdmod):
    # kmd.h: 8 M + 4 bytes per pixel (the (s_i, d_i) pairs and the log-sum-exp plane)
    for N, H, W, sizes in [(1, 1080, 1920, [3, 5, 7, 9, 11, 13]), (2, 64, 96, [3, 5]), (1, 8, 8, [3])]:
        assert kmdmod.backward_workspace_bytes(N, H, W, sizes) == N * H * W * (8 * len(sizes) + 4)


def test_header_is_plain_c99(tmp_path):
    # the boundary is a C ABI: include/kmd.h compiles as strict C99 (no C++ or torch types)
    import shutil
    import subprocess
    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("gcc not found")
    src = tmp_path / "h.c"
    src.write_text('#include "kmd.h"\nint main(void) { kmd_config c; (void)c; return 0; }\n')
    r = subprocess.run([gcc, "-std=c99", "-Wall", "-Wextra", "-Werror", "-pedantic",
                        "-I", os.path.join(ROOT, "include"), "-c", str(src), "-o", str(tmp_path / "h.o")],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
