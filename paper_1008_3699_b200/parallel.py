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


# ---------------------------------------------------------------------------------------------
# One PCG over several slabs.  The arithmetic runs in the library's kernels
# (staged preconditioner, SpMV, fused axpy / dot); this driver only orders the calls, refreshes
# ghost layers between them and sums the ranks' double-double partials in rank order.

def dd_sum(pairs) -> float:
    """Sum (hi, lo) double-double pairs in the given order (TwoSum), rounded once."""
    hi, lo = 0.0, 0.0
    for h, l in pairs:
        t = hi + h
        bp = t - hi
        err = (hi - (t - bp)) + (h - bp)
        hi, lo = t, lo + err + l
    return hi + lo


class LocalComm:
    """All ranks live in this process (virtual slabs, e.g. several Grids on one device)."""

    def __init__(self, grids):
        self.grids = list(grids)

    def exchange(self, views, width):
        exchange_ghosts_local(views, [g.n_local[-1] for g in self.grids], width)

    def allsum(self, pairs):
        return dd_sum(pairs)


class DistComm:
    """One rank per process: ghost layers by torch.distributed point-to-point (NCCL on GPUs),
    reductions by all_gather of the (hi, lo) pairs and a rank-ordered sum on every rank."""

    def __init__(self, grid, group=None, device=None):
        import torch.distributed as dist
        self.grids = [grid]
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        self.group = group
        self.bufs = {}
        self.device = device if device is not None else f"cuda:{grid.device}"

    def exchange(self, views, width):
        exchange_ghosts(views[0], self.grids[0].n_local[-1], self.rank, self.world, self.group, width, self.bufs)

    def allsum(self, pairs):
        import torch
        import torch.distributed as dist
        t = torch.tensor(pairs[0], dtype=torch.float64, device=self.device)
        out = [torch.empty_like(t) for _ in range(self.world)]
        dist.all_gather(out, t, group=self.group)
        return dd_sum([tuple(o.tolist()) for o in out])


def pcg_slabs(comm, precond: int = 2, omega: float = 1.0, pairing: int = 0, rtol: float = 1e-8,
              maxit: int = 10000, msteps: int = 1, theta: float = 0.5, flexible=None):
    """Preconditioned CG from x0 = 0 on the right-hand side SW_B of every slab grid of `comm`
    (same algorithm and stop test as sw_pcg_solve).  msteps > 1 applies the m-step form of the
    preconditioner (sw_set_precond_steps: z_{j+1} = z_j + P^-1 (r - theta A z_j)) through the
    staged solves, sw_apply_A and sw_axpby.  flexible: the Polak-Ribiere beta z+.(r+ - r)/(r.z)
    (None: exactly when the preconditioner is ILU(0) or SSOR with the PAPER pairing, as
    sw_pcg_solve).  Returns (iterations, relres, converged)."""
    import torch

    from . import binding as B
    grids = comm.grids
    dev = f"cuda:{grids[0].device}"
    vecs = (B.X, B.B, B.R, B.Z, B.P, B.Q, B.Y, B.INVD) + ((B.W1, B.W2) if msteps > 1 else ())
    V = {w: [g.view(w) for g in grids] for w in vecs}
    ptr = {w: [t.data_ptr() for t in V[w]] for w in V}
    dd = [torch.zeros(2, dtype=torch.float64, device=dev) for _ in grids]
    if flexible is None:
        flexible = pairing == B.PAIR_PAPER and precond in (B.PC_ILU0, B.PC_SSOR)
    if flexible:                             # r before its update, and r+ - r
        rold = [torch.empty_like(t) for t in V[B.R]]
        rdif = [torch.empty_like(t) for t in V[B.R]]

    def reduce(fn):
        for i, g in enumerate(grids):
            fn(i, g)
        torch.cuda.synchronize()
        return comm.allsum([tuple(d.tolist()) for d in dd])

    for i in range(len(grids)):
        V[B.X][i].zero_()
        V[B.R][i].copy_(V[B.B][i])
    if precond == B.PC_ILU0:
        for g in grids:
            g.ilu0_factor(0)
        comm.exchange(V[B.INVD], 1)
    z = B.R if precond == B.PC_NONE else B.Z

    def apply1(src, dst):                    # dst = P^-1 src, stage by stage
        comm.exchange(V[src], 1)
        for st in range(grids[0].precond_stages(pairing)):
            if st == 1 and pairing == B.PAIR_PAPER:
                comm.exchange(V[B.Y], 1)
            if st >= 2:
                if st == 2:
                    comm.exchange(V[B.Y], 1)
                comm.exchange(V[dst], 2)
            for i, g in enumerate(grids):
                g.precond_apply_stage(precond, st, ptr[src][i], ptr[dst][i], omega, pairing)

    def apply_pc():
        if precond == B.PC_NONE:
            return
        apply1(B.R, B.Z)
        for _ in range(msteps - 1):             # z += P^-1 (r - theta A z)
            comm.exchange(V[B.Z], 1)
            for i, g in enumerate(grids):
                g.apply_A(ptr[B.Z][i], ptr[B.W1][i], dd[i].data_ptr())
                g.axpby(1.0, ptr[B.R][i], -theta, ptr[B.W1][i], ptr[B.W2][i])
            apply1(B.W2, B.W1)
            for i, g in enumerate(grids):
                g.axpby(1.0, ptr[B.Z][i], 1.0, ptr[B.W1][i], ptr[B.Z][i])

    bb = reduce(lambda i, g: g.dot(ptr[B.B][i], ptr[B.B][i], dd[i].data_ptr()))
    bnorm = bb ** 0.5
    if bnorm == 0.0:
        return 0, 0.0, True
    apply_pc()
    rz = reduce(lambda i, g: g.dot(ptr[B.R][i], ptr[z][i], dd[i].data_ptr()))
    for i in range(len(grids)):
        V[B.P][i].copy_(V[z][i])
    relres = 1.0
    for it in range(1, maxit + 1):
        comm.exchange(V[B.P], 1)
        pq = reduce(lambda i, g: g.apply_A(ptr[B.P][i], ptr[B.Q][i], dd[i].data_ptr()))
        alpha = rz / pq
        if flexible:
            for i in range(len(grids)):
                rold[i].copy_(V[B.R][i])
        rr = reduce(lambda i, g: g.axpy2(alpha, ptr[B.X][i], ptr[B.R][i], ptr[B.P][i], ptr[B.Q][i],
                                         dd[i].data_ptr()))
        relres = rr ** 0.5 / bnorm
        if relres < rtol:
            for g in grids:
                g.check()
            return it, relres, True
        if relres != relres:
            raise FloatingPointError("PCG produced NaN")
        apply_pc()
        rzn = reduce(lambda i, g: g.dot(ptr[B.R][i], ptr[z][i], dd[i].data_ptr()))
        if flexible:                         # (r+ - r) rounded first, then z.(r+ - r), as the oracle
            for i, g in enumerate(grids):
                g.axpby(1.0, ptr[B.R][i], -1.0, rold[i].data_ptr(), rdif[i].data_ptr())
            beta = reduce(lambda i, g: g.dot(ptr[z][i], rdif[i].data_ptr(), dd[i].data_ptr())) / rz
        else:
            beta = rzn / rz
        rz = rzn
        for i, g in enumerate(grids):
            g.xpby(ptr[z][i], beta, ptr[B.P][i])
    return maxit, relres, False
