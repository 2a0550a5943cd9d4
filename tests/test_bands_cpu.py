"""Host logic of the multi-GPU row-band split, on CPU: band geometry, and the
halo exchange over torch.distributed with the gloo backend at world size 2 and
3 (each rank's halo rows must equal the corresponding rows of the full frame)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2202_05977_b200 import bands as B

PAPER = [3, 5, 7, 9, 11, 13]


def test_split_rows_geometry():
    bs = B.split_rows(2160, 8, PAPER)
    assert [b.rows for b in bs] == [270] * 8
    assert bs[0].halo_top == 0 and bs[0].halo_bot == 6
    assert bs[-1].halo_top == 6 and bs[-1].halo_bot == 0
    assert all(b.halo_top == 6 and b.halo_bot == 6 for b in bs[1:-1])
    assert sum(b.rows for b in bs) == 2160
    assert all(bs[i].y0 + bs[i].rows == bs[i + 1].y0 for i in range(7))
    one = B.split_rows(100, 1, PAPER)[0]
    assert (one.y0, one.rows, one.halo_top, one.halo_bot) == (0, 100, 0, 0)
    with pytest.raises(ValueError):
        B.split_rows(40, 8, PAPER)   # 5-row bands < r_max = 6


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, H, W, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.Generator().manual_seed(123)
        full = torch.randn((2, 9, H, W), generator=g)       # N=2 frames, 3 + M=6 planes
        band = B.split_rows(H, world, PAPER)[rank]
        buf = torch.full((2, 9, band.buf_rows, W), float("nan"))
        own = full[:, :, band.y0:band.y0 + band.rows]
        buf[:, :, band.halo_top:band.halo_top + band.rows] = own
        B.exchange_halos(buf, band, world)
        ok = torch.equal(buf, B.slice_band(full, band))
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_halo_exchange_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, 60, 17, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    res = dict(q.get(timeout=10) for _ in range(world))
    assert all(p.exitcode == 0 for p in procs)
    assert res == {r: True for r in range(world)}
