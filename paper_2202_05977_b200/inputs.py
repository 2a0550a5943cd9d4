"""Seeded synthetic inputs shaped like the paper's workloads.

This module holds NONE of the method's arithmetic (no unfold, softmax,
filtering or fusion): it only draws random fields.  It is the one module both
the CUDA path's tests/bench and the CPU oracle consume (DESIGN.md "Input
recipe").

Recipe:
  * radiance r_c = L_c * s_c: the 1-spp noisy demodulated HDR irradiance the
    paper filters.  L_c = exp(0.75 * smooth_c) is a smooth
    "clean" signal (~0.1..10), s_c ~ Exp(1) i.i.d. is the 1-spp multiplicative
    noise surrogate, and fireflies multiply a pixel by 100
    with probability 1e-4.
  * importance I_i = 2 * smooth_i + N(0,1): unbounded reals, one map per kernel
    size, typically in [-10, 10].
  * blend logits B_i = 1.5 * smooth'_i + N(0, 0.5^2).
  * smooth = N(0,1) on an (H/32+2) x (W/32+2) grid, bicubic-upsampled to H x W
    and renormalised to zero mean / unit std.
Every frame f of a batch is drawn from its own generator seeded with
``seed + frame_offset + f``, so a batch sharded over ranks is the same set of
frames as the unsharded batch.

Stress distributions (parity only): "uniform40" (I ~ U(-40,40)), "spikes"
(sparse +-40 spikes on the paper recipe), "extreme" (I ~ U(-120,120): forces
the kernels' range fallback), "const" (radiance == 0.5 everywhere).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Sequence

import torch
import torch.nn.functional as F

BASE_SEED = 220205977
PAPER_SIZES = (3, 5, 7, 9, 11, 13)  # k_b = 3, k_s = 2, M = 6

DISTS = ("paper", "uniform40", "spikes", "extreme", "const")


@dataclass
class FrameInputs:
    radiance: torch.Tensor    # [N,3,H,W] fp32
    importance: torch.Tensor  # [N,M,H,W] fp32
    blend: Optional[torch.Tensor]  # [N,M,H,W] fp32, None when M == 1 and no blend wanted


def _smooth(g: torch.Generator, n: int, H: int, W: int, device) -> torch.Tensor:
    gh, gw = H // 32 + 2, W // 32 + 2
    coarse = torch.randn((1, n, gh, gw), generator=g, device=device, dtype=torch.float32)
    f = F.interpolate(coarse, size=(H, W), mode="bicubic", align_corners=False)[0]
    f = f - f.mean(dim=(1, 2), keepdim=True)
    f = f / f.std(dim=(1, 2), keepdim=True).clamp_min(1e-6)
    return f


def _frame(g: torch.Generator, H: int, W: int, M: int, dist: str, with_blend: bool, device):
    # radiance: smooth signal x Exp(1) noise x rare fireflies
    L = torch.exp(0.75 * _smooth(g, 3, H, W, device))
    s = torch.empty((3, H, W), device=device, dtype=torch.float32).exponential_(1.0, generator=g)
    fire = torch.rand((1, H, W), generator=g, device=device) < 1e-4
    rad = L * s * torch.where(fire, 100.0, 1.0)
    if dist == "const":
        rad = torch.full_like(rad, 0.5)
    # importance maps
    if dist in ("paper", "const", "spikes"):
        imp = 2.0 * _smooth(g, M, H, W, device) + torch.randn((M, H, W), generator=g,
                                                              device=device)
        if dist == "spikes":
            u = torch.rand((M, H, W), generator=g, device=device)
            imp = torch.where(u < 5e-3, torch.full_like(imp, 40.0), imp)
            imp = torch.where(u > 1 - 5e-3, torch.full_like(imp, -40.0), imp)
    elif dist == "uniform40":
        imp = (torch.rand((M, H, W), generator=g, device=device) * 2 - 1) * 40.0
    elif dist == "extreme":
        imp = (torch.rand((M, H, W), generator=g, device=device) * 2 - 1) * 120.0
    else:
        raise ValueError(f"unknown dist {dist!r}; expected one of {DISTS}")
    blend = None
    if with_blend:
        blend = 1.5 * _smooth(g, M, H, W, device) + 0.5 * torch.randn((M, H, W), generator=g,
                                                                      device=device)
    return rad.contiguous(), imp.contiguous(), blend


def make_inputs(N: int, H: int, W: int, M: int, seed: int = BASE_SEED, frame_offset: int = 0,
                dist: str = "paper", with_blend: Optional[bool] = None,
                device="cpu") -> FrameInputs:
    """N frames of (radiance, importance, blend) on ``device`` (fp32, planar)."""
    if with_blend is None:
        with_blend = M > 1
    device = torch.device(device)
    rads, imps, blends = [], [], []
    for f in range(N):
        g = torch.Generator(device=device)
        g.manual_seed(seed + frame_offset + f)
        r, i, b = _frame(g, H, W, M, dist, with_blend, device)
        rads.append(r)
        imps.append(i)
        blends.append(b)
    return FrameInputs(torch.stack(rads), torch.stack(imps),
                       torch.stack(blends) if with_blend else None)


def sizes_from(k_b: int = 3, k_s: int = 2, M: int = 6) -> Sequence[int]:
    """k_i = k_b + i * k_s."""
    return tuple(k_b + i * k_s for i in range(M))


def make_albedo(N: int, H: int, W: int, seed: int = BASE_SEED + 7, frame_offset: int = 0,
                device="cpu") -> torch.Tensor:
    """Albedo [N,3,H,W] in (0, 1): a smooth texture (0.05..0.95) with 1% texels
    forced to 0 (the demodulation eps floor)."""
    device = torch.device(device)
    out = []
    for f in range(N):
        g = torch.Generator(device=device)
        g.manual_seed(seed + frame_offset + f)
        a = 0.05 + 0.9 * torch.sigmoid(1.5 * _smooth(g, 3, H, W, device))
        zero = torch.rand((1, H, W), generator=g, device=device) < 0.01
        out.append(torch.where(zero, torch.zeros_like(a), a))
    return torch.stack(out).contiguous()


MR_SIZES = ((3, 5), (3, 5), (3, 5))  # "two filtering kernels with sizes 3 and 5 for each resolution"


@dataclass
class MRInputs:
    radiance: torch.Tensor   # [N,3,H,W]
    importance: list         # per level [N,2,H>>l,W>>l]
    blend: list              # per level [N,2,H>>l,W>>l]
    alpha: list              # per level l < L-1: [N,1,H>>l,W>>l] in [0,1]


def make_mr_inputs(N: int, H: int, W: int, sizes_per_level=MR_SIZES, seed: int = BASE_SEED + 11,
                   device="cpu") -> MRInputs:
    """Inputs of the multi-resolution variant (NEXT row 2): per level the same
    importance / logit recipe as make_inputs, and Eq. 7 blend weights
    alpha = sigmoid(1.5 * smooth + N(0, 0.5^2)) in [0, 1]."""
    L = len(sizes_per_level)
    base = make_inputs(N, H, W, len(sizes_per_level[0]), seed=seed, device=device)
    imps, blends, alphas = [base.importance], [base.blend], []
    for l in range(1, L):
        lv = make_inputs(N, H >> l, W >> l, len(sizes_per_level[l]), seed=seed + 1000 * l,
                         device=device)
        imps.append(lv.importance)
        blends.append(lv.blend)
    device = torch.device(device)
    for l in range(L - 1):
        g = torch.Generator(device=device)
        g.manual_seed(seed + 5000 + l)
        h, w = H >> l, W >> l
        a = torch.stack([torch.sigmoid(1.5 * _smooth(g, 1, h, w, device) +
                                       0.5 * torch.randn((1, h, w), generator=g, device=device))
                         for _ in range(N)])
        alphas.append(a.contiguous())
    return MRInputs(base.radiance, imps, blends, alphas)


@dataclass
class TemporalInputs:
    cur_rad: torch.Tensor     # [N,3,H,W] 1-spp radiance of the current frame
    prev_rad: torch.Tensor    # [N,3,H,W] accumulated radiance of the previous frame
    prev_pos: torch.Tensor    # [N,3,H,W] world positions (scene units)
    prev_nrm: torch.Tensor    # [N,3,H,W] shading normals scaled to [0,1]
    prev_valid: torch.Tensor  # [N,H,W] uint8
    cur_pos: torch.Tensor
    cur_nrm: torch.Tensor
    motion: torch.Tensor      # [N,2,H,W] pixels, channel 0 = x
    pos_tol: float            # 1% of the scene's bounding-box diagonal (SPEC.md DESIGN DECISIONS)


def _scene(u: torch.Tensor, v: torch.Tensor, ph: torch.Tensor):
    """World position and [0,1]-scaled normal of a height-field scene z(u, v)
    seen by an orthographic camera (1 scene unit per pixel)."""
    z = 40.0 + 6.0 * torch.sin(u / 37.0 + ph[0]) * torch.cos(v / 53.0 + ph[1]) + 3.0 * torch.sin((u + v) / 19.0 + ph[2])
    dzdu = (6.0 / 37.0) * torch.cos(u / 37.0 + ph[0]) * torch.cos(v / 53.0 + ph[1]) + (3.0 / 19.0) * torch.cos((u + v) / 19.0 + ph[2])
    dzdv = -(6.0 / 53.0) * torch.sin(u / 37.0 + ph[0]) * torch.sin(v / 53.0 + ph[1]) + (3.0 / 19.0) * torch.cos((u + v) / 19.0 + ph[2])
    n = torch.stack([-dzdu, -dzdv, torch.ones_like(z)])
    n = n / n.norm(dim=0, keepdim=True)
    return torch.stack([u, v, z]), 0.5 * n + 0.5


def make_temporal_inputs(N: int, H: int, W: int, seed: int = BASE_SEED + 23, device="cpu") -> TemporalInputs:
    """NEXT row 4 inputs: a height-field scene under a camera pan of (m0x, m0y)
    pixels per frame plus sub-pixel smooth jitter in the motion vectors; 3% of
    the pixels are disoccluded (current geometry displaced far from the previous
    frame's), 2% have a flipped normal, 0.5% of the history is invalid."""
    device = torch.device(device)
    out = {k: [] for k in ("cur_rad", "prev_rad", "prev_pos", "prev_nrm", "prev_valid", "cur_pos", "cur_nrm",
                           "motion")}
    for f in range(N):
        g = torch.Generator(device=device)
        g.manual_seed(seed + f)
        ph = torch.rand(3, generator=g, device=device) * 6.283
        m0 = (torch.rand(2, generator=g, device=device) * 2 - 1) * 4.0
        yy, xx = torch.meshgrid(torch.arange(H, device=device, dtype=torch.float32),
                                torch.arange(W, device=device, dtype=torch.float32), indexing="ij")
        # the previous frame saw scene point (x' - m0x, y' - m0y) at pixel (x', y')
        prev_pos, prev_nrm = _scene(xx - m0[0], yy - m0[1], ph)
        # pixel p of the current frame shows the point the previous frame had at
        # p + m0, i.e. scene point p
        cur_pos, cur_nrm = _scene(xx, yy, ph)
        motion = m0.view(2, 1, 1) + 0.3 * _smooth(g, 2, H, W, device)
        dis = torch.rand((1, H, W), generator=g, device=device) < 0.03
        cur_pos = torch.where(dis, cur_pos + torch.tensor([0.0, 0.0, 25.0], device=device).view(3, 1, 1), cur_pos)
        flip = torch.rand((1, H, W), generator=g, device=device) < 0.02
        cur_nrm = torch.where(flip, 1.0 - cur_nrm, cur_nrm)
        valid = (torch.rand((H, W), generator=g, device=device) >= 0.005).to(torch.uint8)
        L = torch.exp(0.75 * _smooth(g, 3, H, W, device))
        cur_rad = L * torch.empty((3, H, W), device=device).exponential_(1.0, generator=g)
        prev_rad = L * (1.0 + 0.2 * torch.randn((3, H, W), generator=g, device=device)).clamp_min(0.0)
        for k, v in (("cur_rad", cur_rad), ("prev_rad", prev_rad), ("prev_pos", prev_pos), ("prev_nrm", prev_nrm),
                     ("prev_valid", valid), ("cur_pos", cur_pos), ("cur_nrm", cur_nrm), ("motion", motion)):
            out[k].append(v.contiguous())
    diag = float((W * W + H * H + 20.0 ** 2) ** 0.5)
    return TemporalInputs(**{k: torch.stack(v).contiguous() for k, v in out.items()}, pos_tol=0.01 * diag)
