"""GPU parity at the edges of the unshifted-exp range and under the
paper's invariants, on the TMA kernel (W % 4 == 0, 16-B aligned: the launch
bench.py times).

- Uniform importance I == c with c near ln(FLT_MAX) = 88.72: the box
  denominator sum_q exp(I(q)) overflows (or leaves [1e-30, 1e36]) while the
  numerator may stay finite.  Eq. 3 makes the weights 1/k^2 for any c (a
  uniform map is a box filter, SURVEY.md §8(c) pins), so every such pixel must
  take the exact per-window max-shifted path (reading R13, include/kmd.h
  "Numerics").
- Shift invariance I -> I + c (the importance is "a relative
  value").  Importance values are rounded to multiples of 2^-16
  so that I + 80 is exact in fp32 and the shifted and unshifted inputs define
  the same kernels bit for bit.
- k = 1 is the identity on the TMA kernel's radius-0 code.
"""
import numpy as np
import pytest
import torch

from paper_2202_05977_b200 import inputs as gen
from paper_2202_05977_b200 import kmd
from parity import assert_parity

pytestmark = pytest.mark.gpu

PAPER = list(gen.PAPER_SIZES)


def _gpu(rad, imp, blend, sizes, dev):
    out = kmd.decode_filter_fuse(rad.to(dev), imp.to(dev), None if blend is None else blend.to(dev), sizes)
    torch.cuda.synchronize()
    return out.cpu().numpy()


def _oracle(oracle_mod, rad, imp, blend, sizes):
    return oracle_mod.decode_filter_fuse(rad.numpy(), imp.numpy(), None if blend is None else blend.numpy(), sizes)


@pytest.mark.parametrize("c", [60.0, 84.0, 86.0, 88.0, 88.7])
@pytest.mark.parametrize("sizes", [[3], [13], PAPER])
def test_uniform_high_importance(oracle_mod, cuda_device, c, sizes):
    N, H, W = 1, 54, 104                       # two tile rows, two tile columns, W % 4 == 0
    M = len(sizes)
    g = torch.Generator().manual_seed(int(c * 10) + M)
    rad = 0.05 + 0.55 * torch.rand((N, 3, H, W), generator=g)   # radiance in [0.05, 0.6]
    imp = torch.full((N, M, H, W), c)
    blend = None if M == 1 else torch.randn((N, M, H, W), generator=g)
    out = _gpu(rad, imp, blend, sizes, cuda_device)
    assert kmd.last_kernel() == f"v3-tma-M{M}"
    assert_parity(out, _oracle(oracle_mod, rad, imp, blend, sizes), what=f"I={c} sizes={sizes}")


def test_uniform_high_importance_is_a_box_filter(cuda_device):
    # closed form: a uniform map gives the k x k clamped box mean
    from scipy.ndimage import uniform_filter
    N, H, W, k = 1, 40, 64, 13
    g = torch.Generator().manual_seed(3)
    rad = 0.05 + 0.55 * torch.rand((N, 3, H, W), generator=g)
    out = _gpu(rad, torch.full((N, 1, H, W), 86.0), None, [k], cuda_device)
    ref = np.stack([uniform_filter(rad[0, c].double().numpy(), k, mode="nearest") for c in range(3)])[None]
    assert_parity(out, ref, what="I=86 box")


def _dyadic(t: torch.Tensor) -> torch.Tensor:
    return torch.round(t * 65536.0) / 65536.0  # exact in fp32 after adding 80


@pytest.mark.parametrize("shape,sizes", [((1, 81, 156), PAPER), ((1, 54, 104), [3, 7, 13])])
def test_shift_invariance_I_plus_80(oracle_mod, cuda_device, shape, sizes):
    N, H, W = shape
    inp = gen.make_inputs(N, H, W, len(sizes), seed=91)
    imp = _dyadic(inp.importance)
    shifted = imp + 80.0
    assert torch.equal(shifted - 80.0, imp)
    ref = _oracle(oracle_mod, inp.radiance, imp, inp.blend, sizes)
    base = _gpu(inp.radiance, imp, inp.blend, sizes, cuda_device)
    out = _gpu(inp.radiance, shifted, inp.blend, sizes, cuda_device)
    assert kmd.last_kernel() == f"v3-tma-M{len(sizes)}"
    assert_parity(base, ref, what="I")
    assert_parity(out, ref, what="I + 80")
    # the shifted oracle is the same function: pinned against the unshifted one
    assert_parity(_oracle(oracle_mod, inp.radiance, shifted, inp.blend, sizes), ref, tol=1e-12,
                  what="oracle(I + 80)")


def test_blend_logit_shift_invariance(oracle_mod, cuda_device):
    # softmax(B + c) = softmax(B), including c beyond the exp range
    N, H, W = 1, 54, 104
    inp = gen.make_inputs(N, H, W, 6, seed=93)
    blend = _dyadic(inp.blend)
    ref = _oracle(oracle_mod, inp.radiance, inp.importance, blend, PAPER)
    for c in (-100.0, 80.0, 120.0):
        out = _gpu(inp.radiance, inp.importance, blend + c, PAPER, cuda_device)
        assert_parity(out, ref, what=f"B + {c}")


@pytest.mark.parametrize("shape", [(1, 40, 64), (2, 61, 108)])
def test_k1_identity_on_tma_kernel(cuda_device, shape):
    N, H, W = shape
    inp = gen.make_inputs(N, H, W, 1, seed=95, with_blend=False)
    out = _gpu(inp.radiance, inp.importance, None, [1], cuda_device)
    assert kmd.last_kernel() == "v3-tma-M1"
    assert_parity(out, inp.radiance.double().numpy(), what="k=1")
