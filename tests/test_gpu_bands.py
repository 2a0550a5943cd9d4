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
