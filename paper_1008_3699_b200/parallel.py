"""Multi-GPU slab plumbing: one process per GPU, the slowest grid axis
(y in 2D, z in 3D) split into contiguous slabs of whole tile rows, and the width-2
ghost layers of the iterate exchanged with rank +- 1 before every sweep ("halo points
... renewed (via communication) prior to a new iteration").

The exchange works on any padded tensor whose axis 0 is the slab axis with 2 ghost
layers per side (the device arrays of the C library, viewed through torch, or plain CPU
tensors in the gloo tests); it uses torch.distributed point-to-point ops (NCCL on
GPUs, gloo on CPU).
"""
from __future__ import annotations

from typing import Optional, Tuple

GHOST = 2


def slab_rows(n_tile_rows: int, world: int, rank: int) -> Tuple[int, int]:
    """(first tile row, number of tile rows) of `rank`'s slab; world must divide n_tile_rows."""
    if n_tile_rows % world:
        raise ValueError(f"{world} ranks do not divide {n_tile_rows} tile rows")
    per = n_tile_rows // world
    return rank * per, per


def exchange_ghosts(t, n_local: int, rank: int, world: int, group=None, width: int = GHOST, bufs: Optional[dict] = None):
    """Refresh the ghost layers of padded tensor `t` (axis 0 = slab axis, interior layers at
    [GHOST, GHOST + n_local)) from the neighbouring ranks.  Only `width` layers are sent."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return
    g0 = GHOST
    lo_send = t[g0:g0 + width]
    hi_send = t[g0 + n_local - width:g0 + n_local]
    if bufs is None:
        bufs = {}
    key = (t.data_ptr(), width)
    if key not in bufs:
        bufs[key] = (torch.empty_like(lo_send), torch.empty_like(hi_send))
    lo_recv, hi_recv = bufs[key]
    ops = []
    if rank > 0:
        ops.append(dist.P2POp(dist.isend, lo_send.contiguous(), rank - 1, group))
        ops.append(dist.P2POp(dist.irecv, lo_recv, rank - 1, group))
    if rank < world - 1:
        ops.append(dist.P2POp(dist.isend, hi_send.contiguous(), rank + 1, group))
        ops.append(dist.P2POp(dist.irecv, hi_recv, rank + 1, group))
    for req in dist.batch_isend_irecv(ops):
        req.wait()
    if rank > 0:
        t[g0 - width:g0].copy_(lo_recv)
    if rank < world - 1:
        t[g0 + n_local:g0 + n_local + width].copy_(hi_recv)
