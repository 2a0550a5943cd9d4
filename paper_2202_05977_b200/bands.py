"""Row-band decomposition of one tall frame across ranks.

Host-side geometry plus the halo exchange.  Every output pixel of Eq. 3-5
depends only on its (2 r_max + 1)^2 neighbourhood, so a
frame split into row bands needs exactly one exchange step: each rank receives
r_max rows of the 3 radiance planes and the M importance planes from each
neighbour (blend logits need no halo).  The exchange uses torch.distributed
point-to-point (NCCL over NVLink on GPUs, gloo in the CPU tests); the band
kernel itself is libkmd's kmd_decode_filter_fuse_band.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Sequence

import torch


@dataclass(frozen=True)
class Band:
    rank: int
    y0: int          # first owned global row
    rows: int        # owned rows
    halo_top: int    # rows above y0 held in the input buffers
    halo_bot: int    # rows below y0 + rows held in the input buffers
    H: int           # rows of the whole frame

    @property
    def buf_rows(self) -> int:
        return self.halo_top + self.rows + self.halo_bot

    @property
    def buf_y0(self) -> int:
        return self.y0 - self.halo_top


def rmax_of(sizes: Sequence[int]) -> int:
    return max((int(k) - 1) // 2 for k in sizes)


def split_rows(H: int, G: int, sizes: Sequence[int]) -> List[Band]:
    """Split H rows into G near-equal bands with r_max-row halos (clamped at the
    frame edges, where the kernel clamps instead of reading a neighbour)."""
    if G < 1 or H < G:
        raise ValueError(f"cannot split {H} rows into {G} bands")
    r = rmax_of(sizes)
    bands = []
    for g in range(G):
        y0, y1 = g * H // G, (g + 1) * H // G
        bands.append(Band(g, y0, y1 - y0, min(r, y0), min(r, H - y1), H))
    if G > 1 and min(b.rows for b in bands) < r:
        raise ValueError(f"bands of {min(b.rows for b in bands)} rows are thinner than the "
                         f"halo r_max={r}: a halo would span several ranks")
    return bands


def slice_band(full: torch.Tensor, band: Band) -> torch.Tensor:
    """Rows [y0 - halo_top, y0 + rows + halo_bot) of a [N,C,H,W] tensor (a copy)."""
    return full[:, :, band.buf_y0:band.buf_y0 + band.buf_rows].contiguous()


def exchange_halos(buf: torch.Tensor, band: Band, world: int, group=None) -> None:
    """Fill the halo rows of ``buf`` ([N,C,buf_rows,W], owned rows already set)
    from the neighbouring ranks.  One grouped send/recv step (batch_isend_irecv):
    my first rows go to rank-1 (its bottom halo), my last rows to rank+1 (its
    top halo); neighbours' rows land in my halos."""
    import torch.distributed as dist

    r = band.rank
    ops, recvs = [], []
    own0, own1 = band.halo_top, band.halo_top + band.rows
    if r > 0 and band.halo_top > 0:
        n_up = _peer_halo_bot(band)
        send_up = buf[:, :, own0:own0 + n_up].contiguous()
        recv_top = torch.empty_like(buf[:, :, 0:band.halo_top])
        ops.append(dist.P2POp(dist.isend, send_up, r - 1, group))
        ops.append(dist.P2POp(dist.irecv, recv_top, r - 1, group))
        recvs.append((recv_top, 0))
    if r < world - 1 and band.halo_bot > 0:
        n_down = _peer_halo_top(band)
        send_down = buf[:, :, own1 - n_down:own1].contiguous()
        recv_bot = torch.empty_like(buf[:, :, own1:own1 + band.halo_bot])
        ops.append(dist.P2POp(dist.isend, send_down, r + 1, group))
        ops.append(dist.P2POp(dist.irecv, recv_bot, r + 1, group))
        recvs.append((recv_bot, own1))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    for t, row in recvs:
        buf[:, :, row:row + t.shape[2]].copy_(t)


def _peer_halo_bot(band: Band) -> int:
    # rank-1's bottom halo is min(r_max, H - y0_me) = r_max (my band has >= r_max
    # rows, split_rows checks it), and my halo_top = min(r_max, y0_me) = r_max.
    return band.halo_top


def _peer_halo_top(band: Band) -> int:
    # rank+1's top halo is min(r_max, y0_next) = r_max = my halo_bot.
    return band.halo_bot
