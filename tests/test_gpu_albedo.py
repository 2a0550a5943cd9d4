"""NEXT row 1: albedo remodulation fused into the hot path
(out = Rhat * albedo) and the standalone demodulation /
remodulation ops, vs the fp64 oracle."""
import numpy as np
import pytest
import torch

from paper_2202_05977_b200 import inputs as gen
from paper_2202_05977_b200 import kmd
from parity import assert_parity

pytestmark = pytest.mark.gpu
PAPER = list(gen.PAPER_SIZES)


@pytest.mark.parametrize("H,W,sizes", [(96, 160, PAPER), (37, 45, [3, 5, 7]), (64, 64, [5]), (540, 960, PAPER)])
def test_fused_remodulation_matches_oracle(oracle_mod, cuda_device, H, W, sizes):
    inp = gen.make_inputs(1, H, W, len(sizes), seed=11)
    alb = gen.make_albedo(1, H, W)
    dev = cuda_device
    out = kmd.decode_filter_fuse(inp.radiance.to(dev), inp.importance.to(dev),
                                 None if inp.blend is None else inp.blend.to(dev), sizes,
                                 albedo=alb.to(dev))
    torch.cuda.synchronize()
    if sizes == PAPER:
        assert kmd.last_kernel() == "v3-tma-M6-albedo"
    fused = oracle_mod.decode_filter_fuse(inp.radiance.numpy(), inp.importance.numpy(),
                                          None if inp.blend is None else inp.blend.numpy(), sizes)
    ref = oracle_mod.remodulate(fused, alb.numpy())
    assert_parity(out.cpu().numpy(), ref, what="remod")


def test_remod_with_unit_albedo_is_bitwise_plain(cuda_device):
    inp = gen.make_inputs(1, 120, 200, 6, seed=12, device=cuda_device)
    plain = kmd.decode_filter_fuse(inp.radiance, inp.importance, inp.blend, PAPER)
    ones = torch.ones_like(inp.radiance)
    remod = kmd.decode_filter_fuse(inp.radiance, inp.importance, inp.blend, PAPER, albedo=ones)
    torch.cuda.synchronize()
    assert torch.equal(plain, remod)


def test_demodulate_remodulate_ops(oracle_mod, cuda_device):
    rad = gen.make_inputs(2, 50, 70, 1).radiance
    alb = gen.make_albedo(2, 50, 70)
    d = kmd.demodulate(rad.to(cuda_device), alb.to(cuda_device), eps=1e-3)
    m = kmd.remodulate(d, alb.to(cuda_device))
    torch.cuda.synchronize()
    ref_d = oracle_mod.demodulate(rad.numpy(), alb.numpy(), 1e-3)
    assert_parity(d.cpu().numpy(), ref_d, tol=3e-7, what="demodulate")
    ref_m = oracle_mod.remodulate(d.cpu().numpy().astype(np.float64), alb.numpy())
    assert_parity(m.cpu().numpy(), ref_m, tol=3e-7, what="remodulate")
