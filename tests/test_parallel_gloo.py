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


def _allsum_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = parallel.DistComm(None, device="cpu")
        # rank r contributes the double-double (1 + r, r * 1e-20)
        got = comm.allsum([(1.0 + rank, rank * 1e-20)])
        q.put((rank, got))
    finally:
        dist.destroy_process_group()


def test_distcomm_allsum_is_rank_ordered_and_identical_on_all_ranks():
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_allsum_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = parallel.dd_sum([(1.0 + r, r * 1e-20) for r in range(world)])
    assert all(v == want for v in res.values()) and want == 6.0


def test_dd_sum_is_exact_for_cancellation():
    # (1e16 + 1) - 1e16 lost in plain doubles, kept by the double-double sum
    assert parallel.dd_sum([(1e16, 0.0), (1.0, 0.0), (-1e16, 0.0)]) == 1.0
    assert parallel.dd_sum([]) == 0.0
