"""NEXT row 4: the temporal accumulation pre-pass
(§4.1) on the GPU vs the oracle: the
reprojection / consistency decision (an integer) is compared bit for bit, the
accumulated radiance within the 1e-5 relative bound."""
import numpy as np
import pytest
import torch

from paper_2202_05977_b200 import inputs as gen
from paper_2202_05977_b200 import kmd
from parity import assert_parity

pytestmark = pytest.mark.gpu


def _oracle(oracle_mod, t, **kw):
    return oracle_mod.temporal_accumulate(t.cur_rad.numpy(), t.prev_rad.numpy(), t.prev_pos.numpy(),
                                          t.prev_nrm.numpy(), t.prev_valid.numpy(), t.cur_pos.numpy(),
                                          t.cur_nrm.numpy(), t.motion.numpy(), t.pos_tol, **kw)


def _gpu(t, dev, **kw):
    return kmd.temporal_accumulate(t.cur_rad.to(dev), t.prev_rad.to(dev), t.prev_pos.to(dev),
                                   t.prev_nrm.to(dev), t.prev_valid.to(dev), t.cur_pos.to(dev),
                                   t.cur_nrm.to(dev), t.motion.to(dev), t.pos_tol, **kw)


@pytest.mark.parametrize("N,H,W", [(2, 96, 160), (1, 37, 53), (1, 1080, 1920), (1, 5, 3)])
def test_temporal_matches_oracle(oracle_mod, cuda_device, N, H, W):
    t = gen.make_temporal_inputs(N, H, W, seed=gen.BASE_SEED + 31 + H)
    acc, mask = _gpu(t, cuda_device)
    torch.cuda.synchronize()
    ra, rm = _oracle(oracle_mod, t)
    m = mask.cpu().numpy()
    assert np.array_equal(m, rm), f"mask differs at {np.argwhere(m != rm)[:5]}"
    if H * W > 100:
        assert 0.5 < rm.mean() < 0.99
    assert_parity(acc.cpu().numpy(), ra, what="accum")


def test_temporal_params_and_inplace(oracle_mod, cuda_device):
    t = gen.make_temporal_inputs(1, 64, 96, seed=7)
    for kw in (dict(normal_tol=0.5, alpha=1.0), dict(normal_tol=1.0, alpha=0.05), dict(alpha=0.7)):
        acc, mask = _gpu(t, cuda_device, **kw)
        torch.cuda.synchronize()
        ra, rm = _oracle(oracle_mod, t, **kw)
        assert np.array_equal(mask.cpu().numpy(), rm)
        assert_parity(acc.cpu().numpy(), ra, what=str(kw))
    # accum may alias the current radiance
    cur = t.cur_rad.to(cuda_device)
    ref, _ = _gpu(t, cuda_device)
    out, _ = kmd.temporal_accumulate(cur, t.prev_rad.to(cuda_device), t.prev_pos.to(cuda_device),
                                     t.prev_nrm.to(cuda_device), t.prev_valid.to(cuda_device),
                                     t.cur_pos.to(cuda_device), t.cur_nrm.to(cuda_device),
                                     t.motion.to(cuda_device), t.pos_tol, accum=cur, want_mask=False)
    torch.cuda.synchronize()
    assert out.data_ptr() == cur.data_ptr() and torch.equal(out, ref)


def test_temporal_errors_and_empty(cuda_device):
    t = gen.make_temporal_inputs(1, 16, 16, seed=8)
    d = {k: getattr(t, k).to(cuda_device) for k in ("cur_rad", "prev_rad", "prev_pos", "prev_nrm", "prev_valid",
                                                    "cur_pos", "cur_nrm", "motion")}
    args = [d[k] for k in ("cur_rad", "prev_rad", "prev_pos", "prev_nrm", "prev_valid", "cur_pos", "cur_nrm",
                           "motion")]
    with pytest.raises(kmd.KmdError):
        kmd.temporal_accumulate(*args, pos_tol=0.0)
    with pytest.raises(kmd.KmdError):
        kmd.temporal_accumulate(*args, pos_tol=1.0, alpha=0.0)
    with pytest.raises(kmd.KmdError):  # accum over the previous frame's radiance
        kmd.temporal_accumulate(*args, pos_tol=1.0, accum=d["prev_rad"])
    z3 = torch.empty((0, 3, 16, 16), device=cuda_device)
    z2 = torch.empty((0, 2, 16, 16), device=cuda_device)
    zv = torch.empty((0, 16, 16), device=cuda_device, dtype=torch.uint8)
    acc, mask = kmd.temporal_accumulate(z3, z3, z3, z3, zv, z3, z3, z2, pos_tol=1.0)
    assert acc.shape == (0, 3, 16, 16) and mask.shape == (0, 16, 16)
