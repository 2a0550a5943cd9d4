"""GPU parity: libkmd (CUDA, through the C ABI) vs the fp64 CPU oracle on the
same seeded inputs, element by element, max relative error <= 1e-5
(north_star).  Inputs are generated on the CPU and copied to the
device, so both sides see identical bits."""
import numpy as np
import pytest
import torch

from paper_2202_05977_b200 import inputs as gen
from paper_2202_05977_b200 import kmd
from parity import assert_parity

pytestmark = pytest.mark.gpu

PAPER = list(gen.PAPER_SIZES)


def _run(inp, sizes, dev, logits=True):
    r = inp.radiance.to(dev)
    i = inp.importance.to(dev)
    b = None if inp.blend is None else inp.blend.to(dev)
    out = kmd.decode_filter_fuse(r, i, b, sizes, blend_is_logits=logits)
    torch.cuda.synchronize()
    return out.cpu().numpy()


def _oracle(oracle_mod, inp, sizes, logits=True, **kw):
    b = None if inp.blend is None else inp.blend.numpy()
    return oracle_mod.decode_filter_fuse(inp.radiance.numpy(), inp.importance.numpy(), b,
                                         sizes, blend_is_logits=logits, **kw)


def test_config0_64x64_k5_single_map(oracle_mod, cuda_device):
    # BASELINE.json configs[0]: 64x64, one importance map, k=5, no fusion
    inp = gen.make_inputs(1, 64, 64, 1, with_blend=False)
    assert_parity(_run(inp, [5], cuda_device), _oracle(oracle_mod, inp, [5]), what="64x64 k=5")


def test_config1_720p_paper_set_full_frame(oracle_mod, cuda_device):
    # BASELINE.json configs[1]: 1280x720, {3..13}, fusion -- every pixel checked
    inp = gen.make_inputs(1, 720, 1280, 6)
    assert_parity(_run(inp, PAPER, cuda_device), _oracle(oracle_mod, inp, PAPER),
                  what="720p M=6")


@pytest.mark.parametrize("N,H,W,sizes", [
    (1, 37, 45, [3, 5, 7, 9, 11, 13]),     # ragged tiles both ways, W % 4 != 0
    (3, 19, 70, [3, 7, 11]),                # H < tile height, N > 1
    (2, 33, 33, [1]),                       # k = 1 identity path
    (1, 64, 97, [3, 5]),
    (1, 50, 61, [21]),                      # one large window
    (1, 40, 40, [31]),                      # KMD_MAX_K
    (1, 31, 31, [31, 1, 15, 3, 29, 5, 9, 7]),  # M = 8, unsorted sizes
    (2, 65, 129, [13, 11, 9, 7, 5, 3]),     # paper set, descending order
])
def test_shapes_fuzz(oracle_mod, cuda_device, N, H, W, sizes):
    """Mostly W % 4 != 0 / k > 13 shapes: the v2 and v1 kernels."""
    inp = gen.make_inputs(N, H, W, len(sizes), seed=1000 + H * W)
    out = _run(inp, sizes, cuda_device)
    assert kmd.last_kernel() == ("v1-direct" if max(sizes) > 13 else ("v2-ws" if W % 4 else "v3-tma-M6"))
    assert_parity(out, _oracle(oracle_mod, inp, sizes), what=f"{N}x{H}x{W} {sizes}")


@pytest.mark.parametrize("N,H,W,sizes", [
    (1, 61, 108, [3, 5, 7, 9, 11, 13]),     # M = 6 specialisation, ragged 52x27 tiles both ways
    (1, 27, 52, [3, 5, 7, 9, 11, 13]),      # exactly one tile
    (2, 30, 56, [3, 5]),                    # M = 2 specialisation (MR levels), N > 1
    (1, 83, 200, [3, 7, 11]),               # runtime-M kernel
    (1, 28, 56, [13]),                      # M = 1, the largest TMA window
    (3, 54, 104, [13, 3, 9, 5, 11, 7]),     # M = 6 specialisation, unsorted sizes, N = 3
    (1, 13, 16, [13, 13]),                  # H == k: every row is a border row
    (1, 57, 112, [3, 5, 7, 9, 11, 13, 3, 5]),  # M = 8: the runtime-M kernel
])
def test_tma_kernel_shapes(oracle_mod, cuda_device, N, H, W, sizes):
    """W % 4 == 0: the TMA kernel (kmd_tma.cu) and its specialisations."""
    inp = gen.make_inputs(N, H, W, len(sizes), seed=2000 + H * W)
    out = _run(inp, sizes, cuda_device)
    expect = f"v3-tma-M{len(sizes)}" if len(sizes) <= 6 else "v3-tma"
    assert kmd.last_kernel() == expect
    assert_parity(out, _oracle(oracle_mod, inp, sizes), what=f"tma {N}x{H}x{W} {sizes}")


@pytest.mark.parametrize("dist", ["uniform40", "spikes", "extreme", "const"])
def test_stress_distributions(oracle_mod, cuda_device, dist):
    # "extreme" (I ~ U(-120,120)) forces the per-window max-shift fallback
    inp = gen.make_inputs(1, 96, 160, 6, dist=dist, seed=77)
    assert_parity(_run(inp, PAPER, cuda_device), _oracle(oracle_mod, inp, PAPER), what=dist)


def test_prenormalised_alpha(oracle_mod, cuda_device):
    inp = gen.make_inputs(1, 48, 80, 3)
    a = torch.softmax(inp.blend, dim=1).contiguous()
    inp2 = gen.FrameInputs(inp.radiance, inp.importance, a)
    assert_parity(_run(inp2, [3, 5, 9], cuda_device, logits=False),
                  _oracle(oracle_mod, inp2, [3, 5, 9], logits=False), what="alpha given")


def test_1080p_sampled_in_bench_configuration(oracle_mod, cuda_device):
    # configs[2] at full size, the launch bench.py times: every pixel of a band
    # of rows at the top, the middle and the bottom (borders + interior tiles),
    # plus 4000 random pixels.
    H, W = 1080, 1920
    inp = gen.make_inputs(1, H, W, 6)
    gpu = _run(inp, PAPER, cuda_device)
    for y0, y1 in [(0, 40), (520, 552), (1050, 1080)]:
        ref = _oracle(oracle_mod, inp, PAPER, rows=(y0, y1))
        assert_parity(gpu[:, :, y0:y1], ref, what=f"1080p rows {y0}:{y1}")
    rng = np.random.default_rng(5)
    ys, xs = rng.integers(0, H, 4000), rng.integers(0, W, 4000)
    ref = oracle_mod.decode_filter_fuse_pixels(inp.radiance.numpy(), inp.importance.numpy(),
                                               inp.blend.numpy(), PAPER, np.zeros(4000), ys, xs)
    assert_parity(gpu[0][:, ys, xs].T, ref, what="1080p random pixels")


def test_4k_frame_sampled(oracle_mod, cuda_device):
    # configs[3]'s frame on one GPU: rows at the top / middle / bottom tile rows
    # (2160 = 80 tile rows of 27) and the right-most partial tile column
    H, W = 2160, 3840
    inp = gen.make_inputs(1, H, W, 6, seed=4)
    gpu = _run(inp, PAPER, cuda_device)
    assert kmd.last_kernel() == "v3-tma-M6"
    for y0, y1 in [(0, 30), (1077, 1090), (2140, 2160)]:
        ref = _oracle(oracle_mod, inp, PAPER, rows=(y0, y1))
        assert_parity(gpu[:, :, y0:y1], ref, what=f"4K rows {y0}:{y1}")


def test_batch_of_1080p_frames_sampled(oracle_mod, cuda_device):
    # configs[4] shape (a batch of 1080p frames in one launch), 3 frames sampled
    N, H, W = 4, 1080, 1920
    inp = gen.make_inputs(N, H, W, 6, frame_offset=100)
    gpu = _run(inp, PAPER, cuda_device)
    rng = np.random.default_rng(9)
    n = rng.integers(0, N, 3000)
    ys, xs = rng.integers(0, H, 3000), rng.integers(0, W, 3000)
    ref = oracle_mod.decode_filter_fuse_pixels(inp.radiance.numpy(), inp.importance.numpy(),
                                               inp.blend.numpy(), PAPER, n, ys, xs)
    assert_parity(gpu[n, :, ys, xs], ref, what="batch sampled")


def test_decode_filter_single_size_and_fuse_entry_points(oracle_mod, cuda_device):
    H, W = 57, 83
    inp = gen.make_inputs(1, H, W, 3, seed=4)
    sizes = [3, 9, 13]
    dev = cuda_device
    r = inp.radiance.to(dev)
    filt = torch.stack([kmd.decode_filter(r, inp.importance[:, i:i + 1].contiguous().to(dev), k)
                        for i, k in enumerate(sizes)], dim=1).contiguous()
    torch.cuda.synchronize()
    for i, k in enumerate(sizes):
        ref = oracle_mod.decode_filter_fuse(inp.radiance.numpy(),
                                            inp.importance[:, i:i + 1].numpy(), None, [k])
        assert_parity(filt[:, i].cpu().numpy(), ref, what=f"decode_filter k={k}")
    fused = kmd.fuse(filt, inp.blend.to(dev))
    torch.cuda.synchronize()
    ref = oracle_mod.fuse(filt[0].cpu().numpy().astype(np.float64), inp.blend[0].numpy())
    assert_parity(fused[0].cpu().numpy(), ref, what="kmd_fuse")


def test_host_entry_point_matches_device_path_bitwise(cuda_device):
    N, H, W = 2, 120, 200
    inp = gen.make_inputs(N, H, W, 6, seed=8)
    dev = _run(inp, PAPER, cuda_device)
    out = torch.empty((N, 3, H, W)).pin_memory()
    ws = torch.empty(kmd.host_workspace_bytes(N, H, W, PAPER), dtype=torch.uint8,
                     device=cuda_device)
    kmd.decode_filter_fuse_host(inp.radiance.pin_memory(), inp.importance.pin_memory(),
                                inp.blend.pin_memory(), PAPER, out, ws)
    torch.cuda.synchronize()
    assert np.array_equal(out.numpy(), dev)


def test_empty_batch_is_a_noop(cuda_device):
    z = torch.empty((0, 3, 16, 16), device=cuda_device)
    zi = torch.empty((0, 1, 16, 16), device=cuda_device)
    out = kmd.decode_filter_fuse(z, zi, None, [3])
    assert out.shape == (0, 3, 16, 16)


def test_aliasing_rejected_on_device(cuda_device):
    x = torch.zeros((1, 3, 16, 16), device=cuda_device)
    with pytest.raises(kmd.KmdError, match="ALIAS"):
        kmd.decode_filter_fuse(x, torch.zeros((1, 1, 16, 16), device=cuda_device), None, [3],
                               out=x)


@pytest.mark.parametrize("N,H,W,sizes", [(1, 61, 108, PAPER), (2, 40, 64, [3, 7, 11])])
def test_unaligned_buffers(oracle_mod, cuda_device, N, H, W, sizes):
    # W % 4 == 0 but every buffer starts 4 bytes past a 16-byte boundary: TMA
    # cannot address it, so the v2 kernel (plain loads) runs
    inp = gen.make_inputs(N, H, W, len(sizes), seed=2500 + W)

    def shifted(t):
        flat = torch.empty(t.numel() + 1, device=cuda_device)
        v = flat[1:].view(t.shape)
        v.copy_(t.to(cuda_device))
        return v
    out = shifted(torch.zeros(N, 3, H, W))
    kmd.decode_filter_fuse(shifted(inp.radiance), shifted(inp.importance), shifted(inp.blend), sizes, out=out)
    torch.cuda.synchronize()
    assert kmd.last_kernel() == "v2-ws"
    assert_parity(out.cpu().numpy(), _oracle(oracle_mod, inp, sizes), what=f"unaligned {N}x{H}x{W}")


def test_host_entry_point_back_to_back_calls(cuda_device):
    # consecutive host calls reuse the workspace with their H2D copies streaming
    # back to back (include/kmd.h): every call's output must still be its own
    H, W = 130, 208
    ws = torch.empty(kmd.host_workspace_bytes(1, H, W, PAPER), dtype=torch.uint8, device=cuda_device)
    frames = [gen.make_inputs(1, H, W, 6, seed=300 + f) for f in range(4)]
    outs = [torch.empty((1, 3, H, W)).pin_memory() for _ in frames]
    hin = [(f.radiance.pin_memory(), f.importance.pin_memory(), f.blend.pin_memory()) for f in frames]
    for (r, i, b), o in zip(hin, outs):
        kmd.decode_filter_fuse_host(r, i, b, PAPER, o, ws)
    torch.cuda.synchronize()
    for f, o in zip(frames, outs):
        assert np.array_equal(o.numpy(), _run(f, PAPER, cuda_device))


def test_dependent_launches_read_the_previous_output(cuda_device):
    # The TMA kernel is launched with programmatic dependent launch and may
    # start while the previous kernel on the stream drains: every global access
    # waits on griddepcontrol.wait.  Chain three launches, each reading the
    # previous one's output as its radiance, with nothing in between, and
    # compare with the same chain synchronised after every launch.
    H, W = 96, 160
    frames = [gen.make_inputs(1, H, W, 6, seed=700 + k) for k in range(3)]
    r0 = frames[0].radiance.to(cuda_device)
    ins = [(f.importance.to(cuda_device), f.blend.to(cuda_device)) for f in frames]
    x = r0
    for i, b in ins:  # back to back
        x = kmd.decode_filter_fuse(x, i, b, PAPER)
    chained = x.cpu().numpy()
    y = r0
    for i, b in ins:
        torch.cuda.synchronize()
        y = kmd.decode_filter_fuse(y.clone(), i, b, PAPER)
        torch.cuda.synchronize()
    assert kmd.last_kernel() == "v3-tma-M6"
    assert np.array_equal(chained, y.cpu().numpy())
