"""NEXT row 2: the multi-resolution "Ours MR" reconstruction
(Eq. 7; 3 levels x sizes {3,5}) vs the fp64
oracle.  Eq. 7 subtracts (f - alpha U D f), so the bound is relative to the
magnitude of the terms: |gpu - ref| <= 1e-5 * (|f| + alpha |U D f| + alpha |U c|)."""
import numpy as np
import pytest
import torch

from paper_2202_05977_b200 import inputs as gen
from paper_2202_05977_b200 import kmd
from parity import assert_parity

pytestmark = pytest.mark.gpu


def _dev(t, d):
    return None if t is None else t.to(d)


@pytest.mark.parametrize("N,H,W", [(1, 96, 160), (2, 72, 104), (1, 36, 44), (1, 540, 960), (2, 112, 208),
                                   (3, 56, 112)])
def test_mr_matches_oracle(oracle_mod, cuda_device, N, H, W):
    sizes = [list(s) for s in gen.MR_SIZES]
    mi = gen.make_mr_inputs(N, H, W)
    out = kmd.mr_decode_filter_fuse(mi.radiance.to(cuda_device),
                                    [_dev(t, cuda_device) for t in mi.importance],
                                    [_dev(t, cuda_device) for t in mi.blend],
                                    [_dev(t, cuda_device) for t in mi.alpha], sizes)
    torch.cuda.synchronize()
    # the paper's levels ({3,5} with logits) on TMA-compatible widths take the
    # fused path: 28-row tiles with Eq. 7 in the epilogue (kmd_tma_mr.cu)
    if all((W >> l) % 4 == 0 for l in range(3)):
        assert kmd.last_kernel() == "v3-tma28-mr-cmb"
    ref = oracle_mod.mr_decode_filter_fuse(mi.radiance.numpy(), [t.numpy() for t in mi.importance],
                                           [t.numpy() for t in mi.blend], [t.numpy() for t in mi.alpha],
                                           sizes)
    # scale of the Eq. 7 terms at level 0: the level-0 filtered image bounds them
    f0 = oracle_mod.decode_filter_fuse(mi.radiance.numpy(), mi.importance[0].numpy(),
                                       mi.blend[0].numpy(), sizes[0])
    scale = np.abs(ref) + 2 * np.abs(f0) + 1e-30
    err = np.abs(out.cpu().numpy().astype(np.float64) - ref) / scale
    assert np.all(np.isfinite(out.cpu().numpy()))
    assert err.max() <= 1e-5, err.max()


def test_downsample_and_combine_entry_points(oracle_mod, cuda_device):
    x = gen.make_inputs(2, 40, 52, 1).radiance
    d = kmd.downsample2x2(x.to(cuda_device))
    torch.cuda.synchronize()
    assert_parity(d.cpu().numpy(), oracle_mod.downsample_2x2(x.numpy()), tol=3e-7, what="D")
    fine = gen.make_inputs(1, 40, 52, 1, seed=5).radiance
    coarse = gen.make_inputs(1, 20, 26, 1, seed=6).radiance
    alpha = torch.zeros((1, 1, 40, 52))
    o = kmd.combine_resolutions(fine.to(cuda_device), coarse.to(cuda_device), alpha.to(cuda_device))
    torch.cuda.synchronize()
    assert torch.equal(o.cpu(), fine)       # alpha = 0 -> fine, exactly


@pytest.mark.parametrize("levels,N,H,W", [(2, 1, 64, 88), (4, 1, 96, 160), (1, 2, 40, 48)])
def test_mr_other_level_counts(oracle_mod, cuda_device, levels, N, H, W):
    # 2 levels (no two-level downsample pass), 4 levels (two-level pass + one
    # more 2x2 pass), 1 level (the plain decoder, no auxiliary stream)
    sizes = [[3, 5]] * levels
    mi = gen.make_mr_inputs(N, H, W, sizes_per_level=sizes)
    out = kmd.mr_decode_filter_fuse(mi.radiance.to(cuda_device), [t.to(cuda_device) for t in mi.importance],
                                    [t.to(cuda_device) for t in mi.blend],
                                    [t.to(cuda_device) for t in mi.alpha], sizes)
    torch.cuda.synchronize()
    # the paper's levels ({3,5} with logits) on TMA-compatible widths take the
    # fused path: 28-row tiles with Eq. 7 in the epilogue (kmd_tma_mr.cu)
    if levels > 1 and all((W >> l) % 4 == 0 for l in range(levels)):
        assert kmd.last_kernel() == "v3-tma28-mr-cmb"
    ref = oracle_mod.mr_decode_filter_fuse(mi.radiance.numpy(), [t.numpy() for t in mi.importance],
                                           [t.numpy() for t in mi.blend], [t.numpy() for t in mi.alpha], sizes)
    f0 = oracle_mod.decode_filter_fuse(mi.radiance.numpy(), mi.importance[0].numpy(), mi.blend[0].numpy(),
                                       sizes[0])
    err = np.abs(out.cpu().numpy().astype(np.float64) - ref) / (np.abs(ref) + 2 * np.abs(f0) + 1e-30)
    assert err.max() <= 1e-5, err.max()


def test_mr_inside_cuda_graph_is_bitwise_eager(cuda_device):
    # the coarse levels fork onto an auxiliary stream and join back: the call
    # must be capturable and replay to the same bits
    sizes = [list(s) for s in gen.MR_SIZES]
    mi = gen.make_mr_inputs(1, 108, 208, device=cuda_device)
    ws = torch.empty(kmd.mr_workspace_bytes(1, 108, 208, sizes), dtype=torch.uint8, device=cuda_device)
    eager = kmd.mr_decode_filter_fuse(mi.radiance, mi.importance, mi.blend, mi.alpha, sizes, workspace=ws)
    torch.cuda.synchronize()
    out = torch.empty_like(eager)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        kmd.mr_decode_filter_fuse(mi.radiance, mi.importance, mi.blend, mi.alpha, sizes, out=out, workspace=ws)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    out.zero_()
    with torch.cuda.graph(g):
        kmd.mr_decode_filter_fuse(mi.radiance, mi.importance, mi.blend, mi.alpha, sizes, out=out, workspace=ws)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, eager)


def test_mr_error_paths(cuda_device):
    sizes = [list(s) for s in gen.MR_SIZES]
    mi = gen.make_mr_inputs(1, 96, 160, device=cuda_device)
    ws = torch.empty(kmd.mr_workspace_bytes(1, 96, 160, sizes), dtype=torch.uint8, device=cuda_device)
    # workspace too small
    with pytest.raises(kmd.KmdError):
        kmd.mr_decode_filter_fuse(mi.radiance, mi.importance, mi.blend, mi.alpha, sizes, workspace=ws[:16])
    # H not divisible by 2^(levels-1): 3 levels on 94 rows
    x = gen.make_mr_inputs(1, 96, 160, sizes_per_level=[[3, 5]], device=cuda_device)
    r94 = x.radiance[:, :, :94].contiguous()
    imp = [x.importance[0][:, :, :94].contiguous(), torch.zeros((1, 2, 47, 80), device=cuda_device),
           torch.zeros((1, 2, 23, 40), device=cuda_device)]
    bl = [t.clone() for t in imp]
    al = [torch.zeros((1, 1, 94, 160), device=cuda_device), torch.zeros((1, 1, 47, 80), device=cuda_device)]
    with pytest.raises(kmd.KmdError):
        kmd.mr_decode_filter_fuse(r94, imp, bl, al, sizes)
    # an even kernel size in one level
    with pytest.raises(kmd.KmdError):
        kmd.mr_decode_filter_fuse(mi.radiance, mi.importance, mi.blend, mi.alpha, [[3, 5], [3, 4], [3, 5]])
