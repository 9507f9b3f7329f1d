"""Multi-GPU slab plumbing: one process per GPU, the slowest grid axis
(y in 2D, z in 3D) split into contiguous slabs of whole tile rows, and the width-2
ghost layers of the iterate exchanged with rank +- 1 before every sweep ("halo points
... renewed (via communication) prior to a new iteration").

The exchange works on any padded tensor whose axis 0 is the slab axis with 2 ghost
layers per side (the device arrays of the C library viewed through torch, or plain CPU
tensors in the gloo tests).  ``halo_plan`` says which layers go where; the transports
are torch.distributed point-to-point ops (NCCL on GPUs, gloo on CPU) and, for tests
that emulate several ranks inside one process, plain tensor copies.
"""
from __future__ import annotations

from typing import List, Optional, Sequence, Tuple

GHOST = 2


def slab_rows(n_tile_rows: int, world: int, rank: int) -> Tuple[int, int]:
    """(first tile row, number of tile rows) of `rank`'s slab; world must divide n_tile_rows."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world")
    if n_tile_rows % world:
        raise ValueError(f"{world} ranks do not divide {n_tile_rows} tile rows")
    per = n_tile_rows // world
    return rank * per, per


def halo_plan(n_local: int, rank: int, world: int, width: int = GHOST) -> List[Tuple[int, slice, slice]]:
    """[(peer, send layers, receive layers)] along axis 0 of a padded slab array whose
    interior layers are [GHOST, GHOST + n_local).  The lowest `width` interior layers go
    to rank - 1 and fill its upper ghost layers; the highest go to rank + 1."""
    if not 1 <= width <= GHOST:
        raise ValueError("width must be 1 or 2")
    if n_local < width:
        raise ValueError("slab thinner than the halo")
    g0 = GHOST
    plan = []
    if rank > 0:
        plan.append((rank - 1, slice(g0, g0 + width), slice(g0 - width, g0)))
    if rank < world - 1:
        plan.append((rank + 1, slice(g0 + n_local - width, g0 + n_local), slice(g0 + n_local, g0 + n_local + width)))
    return plan


def exchange_ghosts(t, n_local: int, rank: int, world: int, group=None, width: int = GHOST,
                    bufs: Optional[dict] = None):
    """Refresh the ghost layers of padded tensor `t` from the neighbouring ranks (one
    batched send/recv group; on GPUs this is NCCL over NVLink on the current stream)."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return
    plan = halo_plan(n_local, rank, world, width)
    if bufs is None:
        bufs = {}
    ops, recvs = [], []
    for peer, ss, rs in plan:
        key = (t.data_ptr(), peer, width)
        if key not in bufs:
            bufs[key] = (torch.empty_like(t[ss]), torch.empty_like(t[rs]))
        sbuf, rbuf = bufs[key]
        sbuf.copy_(t[ss])
        ops.append(dist.P2POp(dist.isend, sbuf, peer, group))
        ops.append(dist.P2POp(dist.irecv, rbuf, peer, group))
        recvs.append((rs, rbuf))
    for req in dist.batch_isend_irecv(ops):
        req.wait()
    for rs, rbuf in recvs:
        t[rs].copy_(rbuf)


def exchange_ghosts_local(ts: Sequence, n_locals: Sequence[int], width: int = GHOST):
    """Same exchange for `len(ts)` ranks emulated inside one process (tests): ts[r] is
    rank r's padded array.  All sends are read before any ghost layer is written."""
    world = len(ts)
    moves = []
    for r in range(world):
        for peer, ss, _ in halo_plan(n_locals[r], r, world, width):
            # what r sends to peer lands in peer's receive slice for r
            rs = [p for p in halo_plan(n_locals[peer], peer, world, width) if p[0] == r][0][2]
            moves.append((peer, rs, ts[r][ss].clone()))
    for peer, rs, val in moves:
        ts[peer][rs].copy_(val)
