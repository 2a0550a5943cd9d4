"""Small invocations of every libkmd kernel family, for compute-sanitizer
(SURVEY.md §4 T3): run under memcheck / racecheck / synccheck / initcheck by
scripts/gpu_sanitize.sh.  Each case also checks its result against the
oracle so a silent corruption cannot pass."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402
from paper_2202_05977_b200 import bands as B  # noqa: E402
from paper_2202_05977_b200 import inputs as gen  # noqa: E402
from paper_2202_05977_b200 import kmd  # noqa: E402
from parity import assert_parity  # noqa: E402

PAPER = list(gen.PAPER_SIZES)
dev = torch.device("cuda:0")
which = sys.argv[1:] or ["m1", "m6", "v2", "bands", "bwd", "mr", "bf16", "temporal"]


def fwd(N, H, W, sizes, expect):
    inp = gen.make_inputs(N, H, W, len(sizes), seed=H * W)
    out = kmd.decode_filter_fuse(inp.radiance.to(dev), inp.importance.to(dev),
                                 None if inp.blend is None else inp.blend.to(dev), sizes)
    torch.cuda.synchronize()
    assert kmd.last_kernel() == expect, kmd.last_kernel()
    ref = oracle.decode_filter_fuse(inp.radiance.numpy(), inp.importance.numpy(),
                                    None if inp.blend is None else inp.blend.numpy(), sizes)
    print(f"{expect} {N}x{H}x{W} {sizes}: {assert_parity(out.cpu().numpy(), ref):.2e}")


if "m1" in which:
    fwd(1, 64, 64, [5], "v3-tma-M1")
if "m6" in which:
    fwd(1, 61, 108, PAPER, "v3-tma-M6")
if "v2" in which:
    fwd(1, 37, 45, PAPER, "v2-ws")
if "bands" in which:
    H, W = 120, 104
    inp = gen.make_inputs(1, H, W, 6, seed=7, device=dev)
    whole = kmd.decode_filter_fuse(inp.radiance, inp.importance, inp.blend, PAPER)
    for band in B.split_rows(H, 3, PAPER):
        out = torch.empty((1, 3, band.rows, W), device=dev)
        kw = dict(y0=band.y0, band_rows=band.rows, halo_top=band.halo_top, halo_bot=band.halo_bot,
                  H_global=H, out=out)
        r, i = B.slice_band(inp.radiance, band), B.slice_band(inp.importance, band)
        bl = inp.blend[:, :, band.y0:band.y0 + band.rows].contiguous()
        kmd.decode_filter_fuse_band_part(r, i, bl, PAPER, kmd.BAND_INTERIOR, **kw)
        kmd.decode_filter_fuse_band_part(r, i, bl, PAPER, kmd.BAND_SEAMS, **kw)
        torch.cuda.synchronize()
        assert torch.equal(out, whole[:, :, band.y0:band.y0 + band.rows])
    print("bands 3 x interior + seams: bitwise")
if "bwd" in which:
    N, H, W = 1, 54, 104
    inp = gen.make_inputs(N, H, W, 6, seed=11)
    G = torch.randn((N, 3, H, W), generator=torch.Generator().manual_seed(2))
    ws = torch.empty(kmd.backward_workspace_bytes(N, H, W, PAPER), dtype=torch.uint8, device=dev)
    gi, gb = kmd.decode_filter_fuse_backward(inp.radiance.to(dev), inp.importance.to(dev), inp.blend.to(dev),
                                             G.to(dev), PAPER, workspace=ws)
    torch.cuda.synchronize()
    ri, rb = oracle.backward(inp.radiance.numpy(), inp.importance.numpy(), inp.blend.numpy(), G.numpy(), PAPER)
    e = np.abs(gi.cpu().numpy() - ri).max() / np.abs(ri).max()
    assert e < 1e-5, e
    print(f"backward {kmd.last_kernel()}: normwise {e:.2e}")
if "mr" in which:
    N, H, W = 1, 64, 96
    mi = gen.make_mr_inputs(N, H, W)
    out = kmd.mr_decode_filter_fuse(mi.radiance.to(dev), [t.to(dev) for t in mi.importance],
                                    [t.to(dev) for t in mi.blend], [t.to(dev) for t in mi.alpha],
                                    gen.MR_SIZES)
    torch.cuda.synchronize()
    ref = oracle.mr_decode_filter_fuse(mi.radiance.numpy(), [t.numpy() for t in mi.importance],
                                       [t.numpy() for t in mi.blend], [t.numpy() for t in mi.alpha],
                                       gen.MR_SIZES)
    print(f"mr: {assert_parity(out.cpu().numpy(), ref):.2e}")
if "bf16" in which:
    N, H, W = 1, 54, 104
    inp = gen.make_inputs(N, H, W, 6, seed=13)
    i16, b16 = inp.importance.bfloat16(), inp.blend.bfloat16()
    out = kmd.decode_filter_fuse(inp.radiance.to(dev), i16.to(dev), b16.to(dev), PAPER)
    torch.cuda.synchronize()
    ref = oracle.decode_filter_fuse(inp.radiance.numpy(), i16.float().numpy(), b16.float().numpy(), PAPER)
    print(f"bf16: {assert_parity(out.cpu().numpy(), ref):.2e}")
if "temporal" in which:
    t = gen.make_temporal_inputs(1, 48, 80)
    acc, mask = kmd.temporal_accumulate(*[x.to(dev) for x in (t.cur_rad, t.prev_rad, t.prev_pos, t.prev_nrm,
                                                              t.prev_valid, t.cur_pos, t.cur_nrm, t.motion)],
                                        t.pos_tol)
    torch.cuda.synchronize()
    print("temporal: ok")
print("sanitize cases done")
