"""NEXT row 4's alternative: bf16 importance maps and fusion
logits into the fused hot path (kmd_decode_filter_fuse_bf16).  The operation is
Eq. 3-5 on the bf16 values widened exactly to fp32 (R24), so the
oracle gets the same widened values in fp64 and the fp32 tolerance of
north_star applies unchanged."""
import numpy as np
import pytest
import torch

from paper_2202_05977_b200 import inputs as gen
from paper_2202_05977_b200 import kmd
from parity import assert_parity

pytestmark = pytest.mark.gpu
PAPER = list(gen.PAPER_SIZES)


def _bf16(inp):
    """(importance, blend) rounded to bf16, and the same values widened to fp32."""
    i16 = inp.importance.to(torch.bfloat16)
    b16 = None if inp.blend is None else inp.blend.to(torch.bfloat16)
    return i16, b16, i16.float(), None if b16 is None else b16.float()


def _run16(inp, sizes, dev, logits=True):
    i16, b16, _, _ = _bf16(inp)
    out = kmd.decode_filter_fuse(inp.radiance.to(dev), i16.to(dev), None if b16 is None else b16.to(dev),
                                 sizes, blend_is_logits=logits)
    torch.cuda.synchronize()
    return out


def _oracle(oracle_mod, inp, sizes, logits=True):
    _, _, i32, b32 = _bf16(inp)
    return oracle_mod.decode_filter_fuse(inp.radiance.numpy(), i32.numpy(),
                                         None if b32 is None else b32.numpy(), sizes, blend_is_logits=logits)


@pytest.mark.parametrize("N,H,W,sizes", [
    (1, 96, 160, PAPER),                 # several tiles, ragged last tile row / column
    (2, 37, 48, [3, 5, 7]),              # runtime-M kernel, batch of 2
    (1, 64, 64, [5]),                    # M = 1, no blend
    (1, 20, 56, PAPER),                  # fewer rows than one tile + halo: border rows
    (1, 27, 104, [3, 5, 7, 9]),          # exactly one tile row
])
def test_bf16_matches_oracle(oracle_mod, cuda_device, N, H, W, sizes):
    inp = gen.make_inputs(N, H, W, len(sizes), seed=301)
    out = _run16(inp, sizes, cuda_device)
    assert kmd.last_kernel() == ("v3-tma-bf16-M6" if sizes == PAPER else "v3-tma-bf16")
    assert_parity(out.cpu().numpy(), _oracle(oracle_mod, inp, sizes), what=f"bf16 {N}x{H}x{W} {sizes}")


@pytest.mark.parametrize("dist", ["uniform40", "extreme"])
def test_bf16_stress_distributions(oracle_mod, cuda_device, dist):
    # "extreme" forces the per-window max-shift fallback, which reads the bf16
    # arrays from global memory itself
    inp = gen.make_inputs(1, 96, 160, 6, dist=dist, seed=303)
    assert_parity(_run16(inp, PAPER, cuda_device).cpu().numpy(), _oracle(oracle_mod, inp, PAPER), what=dist)


def test_bf16_prenormalised_alpha(oracle_mod, cuda_device):
    inp = gen.make_inputs(1, 48, 80, 3, seed=304)
    a = torch.softmax(inp.blend, dim=1).contiguous()
    inp2 = gen.FrameInputs(inp.radiance, inp.importance, a)
    assert_parity(_run16(inp2, [3, 5, 9], cuda_device, logits=False).cpu().numpy(),
                  _oracle(oracle_mod, inp2, [3, 5, 9], logits=False), what="bf16 alpha given")


def test_bf16_equals_fp32_path_on_widened_inputs(cuda_device):
    # same arithmetic on the same fp32 values: the two kernels agree bit for bit
    inp = gen.make_inputs(1, 270, 480, 6, seed=305)
    i16, b16, i32, b32 = _bf16(inp)
    r = inp.radiance.to(cuda_device)
    o16 = kmd.decode_filter_fuse(r, i16.to(cuda_device), b16.to(cuda_device), PAPER)
    o32 = kmd.decode_filter_fuse(r, i32.to(cuda_device), b32.to(cuda_device), PAPER)
    torch.cuda.synchronize()
    assert torch.equal(o16, o32)


def test_bf16_1080p_sampled(oracle_mod, cuda_device):
    # the bench's configuration: rows at the top, middle and bottom vs the oracle
    H, W = 1080, 1920
    inp = gen.make_inputs(1, H, W, 6, seed=306)
    out = _run16(inp, PAPER, cuda_device).cpu().numpy()
    _, _, i32, b32 = _bf16(inp)
    for y0 in (0, 532, H - 16):
        ys = slice(max(0, y0 - 6), min(H, y0 + 16 + 6))
        ref = oracle_mod.decode_filter_fuse(inp.radiance[:, :, ys].numpy(), i32[:, :, ys].numpy(),
                                            b32[:, :, ys].numpy(), PAPER)
        # rows whose window lies inside the slice (or touches the frame edge) are exact
        lo = y0 - ys.start
        assert_parity(out[:, :, y0:y0 + 16], ref[:, :, lo:lo + 16], what=f"bf16 1080p rows {y0}")


def test_bf16_errors(cuda_device):
    inp = gen.make_inputs(1, 32, 60, 2, seed=307, device=cuda_device)
    i16, b16 = inp.importance.to(torch.bfloat16), inp.blend.to(torch.bfloat16)
    with pytest.raises(kmd.KmdError) as e:  # W % 8 != 0
        kmd.decode_filter_fuse(inp.radiance, i16, b16, [3, 5])
    assert e.value.status == 4
    inp = gen.make_inputs(1, 32, 64, 2, seed=307, device=cuda_device)
    i16, b16 = inp.importance.to(torch.bfloat16), inp.blend.to(torch.bfloat16)
    with pytest.raises(kmd.KmdError) as e:  # size > 13
        kmd.decode_filter_fuse(inp.radiance, i16, b16, [3, 15])
    assert e.value.status == 2
    with pytest.raises(TypeError):  # mixed dtypes
        kmd.decode_filter_fuse(inp.radiance, i16, inp.blend, [3, 5])
    with pytest.raises(ValueError):
        kmd.decode_filter_fuse(inp.radiance, i16, b16, [3, 5], albedo=torch.ones_like(inp.radiance))
    assert kmd.decode_filter_fuse(inp.radiance[:0], i16[:0], b16[:0], [3, 5]).shape[0] == 0


@pytest.mark.parametrize("N,H,W,sizes", [(2, 120, 200, PAPER), (1, 61, 104, [3, 5, 7]), (1, 48, 64, [5])])
def test_bf16_host_entry_matches_device_path_bitwise(oracle_mod, cuda_device, N, H, W, sizes):
    # kmd_decode_filter_fuse_host_bf16: bf16 importance / logits from pinned
    # host memory, per-band kernels on the same global tile grid -> the device
    # bf16 path bit for bit, and the oracle on the widened values
    inp = gen.make_inputs(N, H, W, len(sizes), seed=4100 + W)
    i16, b16, _, _ = _bf16(inp)
    dev = _run16(inp, sizes, cuda_device).cpu().numpy()
    out = torch.empty((N, 3, H, W)).pin_memory()
    ws = torch.empty(kmd.host_workspace_bytes(N, H, W, sizes), dtype=torch.uint8, device=cuda_device)
    kmd.decode_filter_fuse_host(inp.radiance.pin_memory(), i16.pin_memory(),
                                None if b16 is None else b16.pin_memory(), sizes, out, ws)
    torch.cuda.synchronize()
    assert np.array_equal(out.numpy(), dev)
    assert_parity(out.numpy(), _oracle(oracle_mod, inp, sizes), what=f"bf16 host {N}x{H}x{W}")


def test_bf16_host_entry_rejects_unaligned_width(cuda_device):
    inp = gen.make_inputs(1, 32, 60, 2)
    i16, b16, _, _ = _bf16(inp)
    ws = torch.empty(kmd.host_workspace_bytes(1, 32, 60, [3, 5]), dtype=torch.uint8, device=cuda_device)
    with pytest.raises(kmd.KmdError, match="ALIGN"):
        kmd.decode_filter_fuse_host(inp.radiance, i16, b16, [3, 5], torch.empty((1, 3, 32, 60)), ws)
