"""Row-band kernel (kmd_decode_filter_fuse_band) vs the whole-frame kernel on
ONE GPU: G bands computed in one process from halo-padded slices of the frame
must reproduce the whole-frame output bit for bit (the summation order is a
function of the output pixel only), and match the oracle."""
import numpy as np
import pytest
import torch

from paper_2202_05977_b200 import bands as B
from paper_2202_05977_b200 import inputs as gen
from paper_2202_05977_b200 import kmd
from parity import assert_parity

pytestmark = pytest.mark.gpu
PAPER = list(gen.PAPER_SIZES)


@pytest.mark.parametrize("H,W,G", [(1080, 1920, 2), (2160, 3840, 8), (200, 333, 4), (77, 64, 3)])
def test_bands_bitwise_equal_whole_frame(cuda_device, H, W, G):
    inp = gen.make_inputs(1, H, W, 6, seed=31 + G, device=cuda_device)
    whole = kmd.decode_filter_fuse(inp.radiance, inp.importance, inp.blend, PAPER)
    for band in B.split_rows(H, G, PAPER):
        out = kmd.decode_filter_fuse_band(
            B.slice_band(inp.radiance, band), B.slice_band(inp.importance, band),
            inp.blend[:, :, band.y0:band.y0 + band.rows].contiguous(), PAPER,
            y0=band.y0, band_rows=band.rows, halo_top=band.halo_top, halo_bot=band.halo_bot,
            H_global=H)
        torch.cuda.synchronize()
        assert torch.equal(out, whole[:, :, band.y0:band.y0 + band.rows]), f"band {band}"


def test_band_matches_oracle(oracle_mod, cuda_device):
    H, W = 150, 96
    inp = gen.make_inputs(1, H, W, 6, seed=3)
    band = B.split_rows(H, 3, PAPER)[1]
    dev = cuda_device
    out = kmd.decode_filter_fuse_band(
        B.slice_band(inp.radiance, band).to(dev), B.slice_band(inp.importance, band).to(dev),
        inp.blend[:, :, band.y0:band.y0 + band.rows].contiguous().to(dev), PAPER,
        y0=band.y0, band_rows=band.rows, halo_top=band.halo_top, halo_bot=band.halo_bot,
        H_global=H)
    torch.cuda.synchronize()
    ref = oracle_mod.decode_filter_fuse(inp.radiance.numpy(), inp.importance.numpy(),
                                        inp.blend.numpy(), PAPER, rows=(band.y0, band.y0 + band.rows))
    assert_parity(out.cpu().numpy(), ref, what="band vs oracle")


@pytest.mark.parametrize("sizes,W", [([21, 5], 96), ([3, 5, 7], 90)])
def test_bands_bitwise_other_kernels(cuda_device, sizes, W):
    # the v1 kernel (k > 13) and the v2 kernel (W % 4 != 0) keep the same
    # band-invariance: their summation order depends on the global tile grid only
    H = 160
    inp = gen.make_inputs(1, H, W, len(sizes), seed=91, device=cuda_device)
    whole = kmd.decode_filter_fuse(inp.radiance, inp.importance, inp.blend, sizes)
    kind = kmd.last_kernel()
    assert kind == ("v1-direct" if max(sizes) > 13 else "v2-ws")
    for band in B.split_rows(H, 3, sizes):
        out = kmd.decode_filter_fuse_band(
            B.slice_band(inp.radiance, band), B.slice_band(inp.importance, band),
            inp.blend[:, :, band.y0:band.y0 + band.rows].contiguous(), sizes,
            y0=band.y0, band_rows=band.rows, halo_top=band.halo_top, halo_bot=band.halo_bot,
            H_global=H)
        torch.cuda.synchronize()
        assert kmd.last_kernel() == kind
        assert torch.equal(out, whole[:, :, band.y0:band.y0 + band.rows]), f"band {band}"


# --------------------------------------------------------------------------
# the band interior runs while the halo rows are in flight,
# the seams after.  Single-GPU emulation: the halo rows hold NaN garbage while
# the interior part runs, then the true rows; interior + seams must equal the
# whole-frame output bit for bit (the interior never read a halo row).
@pytest.mark.parametrize("H,W,G", [(2160, 3840, 2), (2160, 3840, 4), (2160, 3840, 8), (540, 960, 8),
                                   (200, 336, 3)])
def test_band_interior_then_seams_bitwise(cuda_device, H, W, G):
    inp = gen.make_inputs(1, H, W, 6, seed=41 + G, device=cuda_device)
    whole = kmd.decode_filter_fuse(inp.radiance, inp.importance, inp.blend, PAPER)
    for band in B.split_rows(H, G, PAPER):
        rad = B.slice_band(inp.radiance, band)
        imp = B.slice_band(inp.importance, band)
        good_r, good_i = rad.clone(), imp.clone()
        for t in (rad, imp):  # halo rows not yet received
            t[:, :, :band.halo_top] = float("nan")
            t[:, :, band.halo_top + band.rows:] = float("nan")
        bl = inp.blend[:, :, band.y0:band.y0 + band.rows].contiguous()
        out = torch.full((1, 3, band.rows, W), float("nan"), device=cuda_device)
        kw = dict(y0=band.y0, band_rows=band.rows, halo_top=band.halo_top, halo_bot=band.halo_bot,
                  H_global=H, out=out)
        kmd.decode_filter_fuse_band_part(rad, imp, bl, PAPER, kmd.BAND_INTERIOR, **kw)
        torch.cuda.synchronize()
        rad.copy_(good_r)
        imp.copy_(good_i)
        kmd.decode_filter_fuse_band_part(rad, imp, bl, PAPER, kmd.BAND_SEAMS, **kw)
        torch.cuda.synchronize()
        assert torch.equal(out, whole[:, :, band.y0:band.y0 + band.rows]), f"band {band}"


def test_band_interior_covers_most_rows(cuda_device):
    # the interior part writes every row farther than r_max (+ the tile grid)
    # from a seam: at G = 8 on 4K, rows 27..242 of a 270-row band at least
    H, W, G = 2160, 3840, 8
    inp = gen.make_inputs(1, H, W, 6, seed=5, device=cuda_device)
    band = B.split_rows(H, G, PAPER)[3]
    out = torch.full((1, 3, band.rows, W), float("nan"), device=cuda_device)
    kmd.decode_filter_fuse_band_part(B.slice_band(inp.radiance, band), B.slice_band(inp.importance, band),
                                     inp.blend[:, :, band.y0:band.y0 + band.rows].contiguous(), PAPER,
                                     kmd.BAND_INTERIOR, y0=band.y0, band_rows=band.rows,
                                     halo_top=band.halo_top, halo_bot=band.halo_bot, H_global=H, out=out)
    torch.cuda.synchronize()
    written = ~torch.isnan(out[0, 0, :, 0])
    assert written[27:243].all()
    assert not written[:6].any() and not written[-6:].any()


def test_nccl_world_size_1_halo_exchange_self_loop(cuda_device):
    # the C entry point on a real one-rank NCCL communicator: a rank that is its
    # own neighbour receives its first owned rows into the top halo and its last
    # owned rows into the bottom halo (include/kmd.h, kmd_halo_exchange)
    comm = kmd.Comm(kmd.nccl_unique_id(), 1, 0)
    try:
        rows, W, h = 40, 64, 6
        planes = [torch.randn((h + rows + h, W), device=cuda_device) for _ in range(9)]
        want = []
        for p in planes:
            w = p.clone()
            w[:h] = p[h:2 * h]
            w[h + rows:] = p[rows:h + rows]
            want.append(w)
        kmd.halo_exchange(comm, planes, rows, h, 0, 0)
        torch.cuda.synchronize()
        for p, w in zip(planes, want):
            assert torch.equal(p, w)
    finally:
        comm.destroy()


def test_nccl_world_size_1_band_step(cuda_device):
    # kmd_band_step with the exchange on its own stream: self-loop neighbours
    # on a one-rank communicator give a band whose halos hold its own edge rows;
    # the result must equal the band call on buffers holding the same halos
    comm = kmd.Comm(kmd.nccl_unique_id(), 1, 0)
    try:
        H, W, h = 540, 960, 6
        band = B.Band(0, 108, 270, h, h, H)
        inp = gen.make_inputs(1, H, W, 6, seed=17, device=cuda_device)
        rad = B.slice_band(inp.radiance, band)
        imp = B.slice_band(inp.importance, band)
        bl = inp.blend[:, :, band.y0:band.y0 + band.rows].contiguous()
        ref_r, ref_i = rad.clone(), imp.clone()
        for t in (ref_r, ref_i):
            t[:, :, :h] = t[:, :, h:2 * h]
            t[:, :, h + band.rows:] = t[:, :, band.rows:h + band.rows]
        ref = kmd.decode_filter_fuse_band(ref_r, ref_i, bl, PAPER, y0=band.y0, band_rows=band.rows,
                                          halo_top=h, halo_bot=h, H_global=H)
        out = torch.empty_like(ref)
        side = torch.cuda.Stream(cuda_device)
        kmd.band_step(comm, rad, imp, bl, PAPER, out, y0=band.y0, band_rows=band.rows, halo=h,
                      peer_up=0, peer_down=0, H_global=H, comm_stream=side)
        torch.cuda.synchronize()
        assert torch.equal(rad, ref_r) and torch.equal(imp, ref_i)
        assert torch.equal(out, ref)
    finally:
        comm.destroy()


def test_band_step_without_neighbours_is_the_whole_frame(cuda_device):
    H, W = 200, 320
    inp = gen.make_inputs(1, H, W, 6, seed=23, device=cuda_device)
    whole = kmd.decode_filter_fuse(inp.radiance, inp.importance, inp.blend, PAPER)
    out = torch.empty_like(whole)
    kmd.band_step(None, inp.radiance.clone(), inp.importance.clone(), inp.blend, PAPER, out, y0=0,
                  band_rows=H, halo=6, peer_up=-1, peer_down=-1, H_global=H)
    torch.cuda.synchronize()
    assert torch.equal(out, whole)
