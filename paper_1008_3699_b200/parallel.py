"""Multi-GPU slab plumbing: one process per GPU, the slowest grid axis
(y in 2D, z in 3D) split into contiguous slabs of whole tile rows, and the width-2
ghost layers of the iterate exchanged with rank +- 1 before every sweep ("halo points
... renewed (via communication) prior to a new iteration").

The library does this itself when its grid has a communicator (sw_comm: NCCL, or a HOST
transport below); ``exchange_ghosts`` / ``exchange_ghosts_local`` are the caller-side
equivalents for grids without one (the staged C calls), on any padded tensor whose axis 0
is the slab axis with 2 ghost layers per side.  ``halo_plan`` says which layers go where.
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


# ---------------------------------------------------------------------------------------------
# Communicators for the library's own multi-rank path (sw_comm, include/sweep.h).  With one the
# library exchanges the ghost layers and sums the reductions itself (NCCL on GPUs, one process per
# GPU); these helpers only create it.  The HOST transports move the staged layers for processes or
# threads that share one GPU (tests): the library calls them with pinned host buffers.

def nccl_comm(device: int, group=None):
    """NCCL communicator of the torch.distributed group's ranks (rank 0 makes the unique id and
    broadcasts it through the group)."""
    import torch.distributed as dist

    from . import binding as B
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    obj = [B.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return B.Comm.nccl(obj[0], rank, world, device)


class GlooTransport:
    """HOST transport over a torch.distributed (gloo) group: one process per rank."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.group = group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)

    def exchange(self, send_lo, recv_lo, send_hi, recv_hi):
        import torch
        import torch.distributed as dist
        ops = []
        if send_lo is not None:
            ops.append(dist.P2POp(dist.isend, torch.from_numpy(send_lo), self.rank - 1, self.group))
            ops.append(dist.P2POp(dist.irecv, torch.from_numpy(recv_lo), self.rank - 1, self.group))
        if send_hi is not None:
            ops.append(dist.P2POp(dist.isend, torch.from_numpy(send_hi), self.rank + 1, self.group))
            ops.append(dist.P2POp(dist.irecv, torch.from_numpy(recv_hi), self.rank + 1, self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()

    def allgather(self, send, recv):
        import torch
        import torch.distributed as dist
        out = [torch.empty(send.size, dtype=torch.uint8) for _ in range(self.world)]
        dist.all_gather(out, torch.from_numpy(send.copy()), group=self.group)
        recv[:] = torch.cat(out).numpy()


class ThreadHub:
    """In-process HOST transport: `world` ranks as threads of one process (each drives its own
    grid on its own stream); every exchange / all-gather is a barrier-separated swap."""

    def __init__(self, world: int):
        import threading
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots = [None] * world

    def endpoint(self, rank: int):
        return _ThreadEndpoint(self, rank)


class _ThreadEndpoint:
    def __init__(self, hub: ThreadHub, rank: int):
        self.hub, self.rank = hub, rank

    def exchange(self, send_lo, recv_lo, send_hi, recv_hi):
        h, r = self.hub, self.rank
        h.slots[r] = (None if send_lo is None else send_lo.copy(), None if send_hi is None else send_hi.copy())
        h.barrier.wait()
        if recv_lo is not None:
            recv_lo[:] = h.slots[r - 1][1]          # rank - 1 sends its upper layers
        if recv_hi is not None:
            recv_hi[:] = h.slots[r + 1][0]          # rank + 1 sends its lower layers
        h.barrier.wait()

    def allgather(self, send, recv):
        h, r = self.hub, self.rank
        h.slots[r] = send.copy()
        h.barrier.wait()
        n = send.size
        for q in range(h.world):
            recv[q * n:(q + 1) * n] = h.slots[q]
        h.barrier.wait()


def host_comm(rank: int, world: int, transport):
    from . import binding as B
    return B.Comm.host(rank, world, transport)
