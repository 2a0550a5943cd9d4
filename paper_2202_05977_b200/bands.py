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
    from the neighbouring ranks in one grouped send/recv step
    (batch_isend_irecv), posted directly on each plane's halo / edge rows (a
    contiguous [rows, W] block of the plane; no staging copies).  Same order
    and meaning as libkmd's kmd_halo_exchange (include/kmd.h), which does this
    over NCCL on GPUs: my first rows go to rank-1 (its bottom halo), my last
    rows to rank+1 (its top halo); neighbours' rows land in my halos."""
    import torch.distributed as dist

    assert buf.is_contiguous()
    r = band.rank
    own0, own1 = band.halo_top, band.halo_top + band.rows
    up = r > 0 and band.halo_top > 0
    down = r < world - 1 and band.halo_bot > 0
    ops = []
    N, C = buf.shape[0], buf.shape[1]
    for n in range(N):
        for c in range(C):
            pl = buf[n, c]
            if up:
                ops.append(dist.P2POp(dist.irecv, pl[0:band.halo_top], r - 1, group))
            if down:
                ops.append(dist.P2POp(dist.irecv, pl[own1:own1 + band.halo_bot], r + 1, group))
            if up:
                ops.append(dist.P2POp(dist.isend, pl[own0:own0 + _peer_halo_bot(band)], r - 1, group))
            if down:
                ops.append(dist.P2POp(dist.isend, pl[own1 - _peer_halo_top(band):own1], r + 1, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()


def make_comm(group=None):
    """libkmd NCCL communicator over the ranks of ``group`` (torch.distributed
    initialised): rank 0's kmd_nccl_unique_id is broadcast to every rank."""
    import torch.distributed as dist

    from . import kmd
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    uid = [kmd.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0, group=group)
    return kmd.Comm(uid[0], world, rank)


def _peer_halo_bot(band: Band) -> int:
    # rank-1's bottom halo is min(r_max, H - y0_me) = r_max (my band has >= r_max
    # rows, split_rows checks it), and my halo_top = min(r_max, y0_me) = r_max.
    return band.halo_top


def _peer_halo_top(band: Band) -> int:
    # rank+1's top halo is min(r_max, y0_next) = r_max = my halo_bot.
    return band.halo_bot
