"""Multi-rank host logic on CPU (gloo, world_size 2 and 3): the slab split and the width-2
ghost-layer exchange that precedes every decomposed sweep on N GPUs (PAPER:828-833,
SURVEY §8(e)).  The check: after the exchange every rank's padded array equals the
corresponding window of the single global array, i.e. each sweep sees exactly the old
values a single-GPU sweep would read."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1008_3699_b200 import parallel

GH = parallel.GHOST


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _global_field(n_rows, width):
    # distinct value per (layer, column); zero ghost layers outside the domain (Dirichlet)
    g = torch.zeros(n_rows + 2 * GH, width, dtype=torch.float64)
    g[GH:GH + n_rows] = torch.arange(n_rows * width, dtype=torch.float64).reshape(n_rows, width) + 1.0
    return g


def _slab(gfield, rank, world, tile, n_rows):
    r0, nr = parallel.slab_rows(n_rows // tile, world, rank)
    lo, n_local = r0 * tile, nr * tile
    t = torch.full((n_local + 2 * GH, gfield.shape[1]), -7.0, dtype=torch.float64)
    t[GH:GH + n_local] = gfield[GH + lo:GH + lo + n_local]
    # physical boundary ghosts are zero on the ends of the domain
    if rank == 0:
        t[:GH] = 0.0
    if rank == world - 1:
        t[GH + n_local:] = 0.0
    return t, lo, n_local


def _worker(rank, world, port, n_rows, tile, width, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = _global_field(n_rows, 5)
        t, lo, n_local = _slab(g, rank, world, tile, n_rows)
        bufs = {}
        for _ in range(2):       # twice: buffers are reused
            parallel.exchange_ghosts(t, n_local, rank, world, width=width, bufs=bufs)
        want = g[lo:lo + n_local + 2 * GH].clone()
        if width == 1:           # only the innermost ghost layer is refreshed
            if rank > 0:
                want[0] = -7.0
            if rank < world - 1:
                want[-1] = -7.0
        q.put((rank, bool(torch.equal(t, want))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n_rows,tile,width", [(2, 16, 4, 2), (3, 24, 4, 2), (2, 8, 2, 1)])
def test_gloo_exchange_reproduces_global_window(world, n_rows, tile, width):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_rows, tile, width, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(res.values()), res


def test_local_exchange_matches_global_window():
    n_rows, tile, world = 24, 4, 3
    g = _global_field(n_rows, 3)
    slabs = [_slab(g, r, world, tile, n_rows) for r in range(world)]
    parallel.exchange_ghosts_local([s[0] for s in slabs], [s[2] for s in slabs])
    for t, lo, n_local in slabs:
        assert torch.equal(t, g[lo:lo + n_local + 2 * GH])


def test_slab_rows_and_plan_validation():
    assert parallel.slab_rows(256, 8, 3) == (96, 32)
    with pytest.raises(ValueError):
        parallel.slab_rows(10, 4, 0)
    assert parallel.halo_plan(8, 0, 1) == []
    plan = parallel.halo_plan(8, 1, 3)
    assert [p[0] for p in plan] == [0, 2]
    assert plan[0][1] == slice(2, 4) and plan[0][2] == slice(0, 2)
    assert plan[1][1] == slice(8, 10) and plan[1][2] == slice(10, 12)
    with pytest.raises(ValueError):
        parallel.halo_plan(1, 0, 2)


def _transport_exchange(tr, t, n_local, width, rank, world):
    """What the library's HOST transport does with a padded slab array (csrc/comm.cuh
    comm_exchange): stage the w lowest / highest interior layers, call the transport, write its
    received bytes into the ghost layers."""
    import numpy as np
    a = t.numpy()
    lo, hi = rank > 0, rank < world - 1
    s_lo = np.ascontiguousarray(a[GH:GH + width]).view(np.uint8).ravel() if lo else None
    s_hi = np.ascontiguousarray(a[GH + n_local - width:GH + n_local]).view(np.uint8).ravel() if hi else None
    r_lo = np.empty_like(s_lo) if lo else None
    r_hi = np.empty_like(s_hi) if hi else None
    tr.exchange(s_lo, r_lo, s_hi, r_hi)
    if lo:
        a[GH - width:GH] = r_lo.view(np.float64).reshape(width, -1)
    if hi:
        a[GH + n_local:GH + n_local + width] = r_hi.view(np.float64).reshape(width, -1)


def _gloo_transport_worker(rank, world, port, n_rows, tile, width, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import numpy as np
        tr = parallel.GlooTransport()
        g = _global_field(n_rows, 5)
        t, lo, n_local = _slab(g, rank, world, tile, n_rows)
        for _ in range(2):
            _transport_exchange(tr, t, n_local, width, rank, world)
        want = g[lo:lo + n_local + 2 * GH].clone()
        if width == 1:
            if rank > 0:
                want[0] = -7.0
            if rank < world - 1:
                want[-1] = -7.0
        send = np.array([1.0 + rank, rank * 1e-20]).view(np.uint8)
        recv = np.empty(send.size * world, dtype=np.uint8)
        tr.allgather(send, recv)
        gathered = recv.view(np.float64).tolist()
        q.put((rank, (bool(torch.equal(t, want)), gathered)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n_rows,tile,width", [(2, 16, 4, 2), (3, 24, 4, 2), (2, 8, 2, 1)])
def test_gloo_host_transport_exchange_and_allgather(world, n_rows, tile, width):
    """parallel.GlooTransport, the multi-process HOST transport of sw_comm_init_host: after the
    exchange every rank's padded slab equals its window of the global array; the all-gather
    returns every rank's bytes in rank order on every rank."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_transport_worker, args=(r, world, port, n_rows, tile, width, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [v for r in range(world) for v in (1.0 + r, r * 1e-20)]
    assert all(ok and gathered == want for ok, gathered in res.values()), res


def test_thread_hub_transport_exchange_and_allgather():
    """parallel.ThreadHub, the in-process HOST transport (ranks as threads): same properties."""
    import threading

    import numpy as np
    n_rows, tile, world, width = 24, 4, 3, 2
    g = _global_field(n_rows, 3)
    slabs = [_slab(g, r, world, tile, n_rows) for r in range(world)]
    hub = parallel.ThreadHub(world)
    gathered = [None] * world

    def body(r):
        ep = hub.endpoint(r)
        t, lo, n_local = slabs[r]
        _transport_exchange(ep, t, n_local, width, r, world)
        recv = np.empty(8 * world, dtype=np.uint8)
        ep.allgather(np.array([float(r)]).view(np.uint8), recv)
        gathered[r] = recv.view(np.float64).tolist()
    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for t, lo, n_local in slabs:
        assert torch.equal(t, g[lo:lo + n_local + 2 * GH])
    assert all(v == [0.0, 1.0, 2.0] for v in gathered)
