"""Decomposed fast sweeping for |grad u| = f through the C ABI (k_eik2) against the
oracle's or_eik_sweep: every pass bitwise (single grid and slabs with the library's communicator),
the number of nodes a pass changes, convergence to the oracle's fixed point, and argument checks."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_1008_3699_b200 import binding as B, gen
from tests.slab_helpers import local_part, run_threads

pytestmark = pytest.mark.gpu
INF = np.inf


def slowness(shape, seed):
    return 0.5 + 1.5 * gen.unit(seed, gen.STREAM_TEST, int(np.prod(shape))).reshape(shape)


def initial(shape, seed):
    """+inf with a few sources (0) and some finite old values (so every branch is exercised)."""
    r = gen.unit(seed, gen.STREAM_X0, int(np.prod(shape))).reshape(shape)
    u = np.where(r < 0.01, 0.0, INF)
    u = np.where((r > 0.6) & (r < 0.7), 50.0 * r, u)
    u[shape[0] // 3, shape[1] // 2] = 0.0
    return u


def eik_grid(n, tile, f, h, rank=0, nranks=1, comm=None):
    g = B.Grid(2, n).decompose(tile, rank, nranks, comm)
    g.set_slowness(local_part(g, f) if nranks > 1 else f, h)
    return g


CASES = [((128, 96), (64, 32)), ((130, 66), (26, 22)), ((64, 64), (64, 64)), ((40, 36), (8, 9)),
         ((256, 256), (64, 64)), ((48, 20), (1, 2)), ((33, 7), (3, 7))]


@pytest.mark.parametrize("n,tile", CASES)
def test_eikonal_passes_match_oracle(n, tile):
    pb = O.tiled(n, tile)
    f = slowness(pb.shape, 1)
    h = 1.0 / n[0]
    u = initial(pb.shape, 2)
    g = eik_grid(n, tile, f, h)
    g.set_vector(B.X, u)
    ph = 0
    for k in range(6):
        un = O.eik_sweep(pb, f, h, u, phase=k)
        ph = g.eikonal_sweep(1, ph)
        got = g.get_vector(B.X)
        assert np.array_equal(got, un), k
        assert g.eikonal_changes() == int(np.sum(un != u)), k
        u = un
    g.check()


@pytest.mark.parametrize("n,tile", [((96, 80), (32, 16)), ((64, 64), (16, 16))])
def test_eikonal_converges_to_the_oracle_fixed_point(n, tile):
    pb = O.tiled(n, tile)
    f = slowness(pb.shape, 3)
    h = 0.01
    u = np.full(pb.shape, INF)
    u[5, 7] = 0.0
    u[-3, -9] = 0.0
    g = eik_grid(n, tile, f, h)
    g.set_vector(B.X, u)
    ph, k = 0, 0
    while True:
        ph = g.eikonal_sweep(4, ph)
        if g.eikonal_changes() == 0:
            break
        assert ph < 400
    for k in range(ph):
        u = O.eik_sweep(pb, f, h, u, phase=k)
    assert np.array_equal(g.get_vector(B.X), u)
    assert np.array_equal(O.eik_sweep(pb, f, h, u, phase=ph), u)      # the oracle's fixed point too


@pytest.mark.parametrize("n,tile,nranks", [((128, 256), (32, 32), 2), ((96, 192), (16, 16), 4), ((64, 96), (64, 8), 3)])
def test_eikonal_over_slabs_matches_oracle(n, tile, nranks):
    """The library's multi-rank path (communicator, exchange behind the interior rows): bitwise."""
    pb = O.tiled(n, tile)
    f = slowness(pb.shape, 4)
    h = 1.0 / n[1]
    u0 = initial(pb.shape, 5)
    nsw = 7

    def rank_fn(r, comm):
        s = torch.cuda.Stream().cuda_stream
        g = eik_grid(n, tile, f, h, r, nranks, comm)
        g.set_vector(B.X, local_part(g, u0), stream=s)
        g.eikonal_sweep(nsw, 0, stream=s)
        return g.get_vector(B.X, stream=s), g.eikonal_changes(stream=s)
    res = run_threads(nranks, rank_fn)
    want_prev = u0
    for k in range(nsw):
        want = O.eik_sweep(pb, f, h, want_prev, phase=k)
        if k < nsw - 1:
            want_prev = want
    assert np.array_equal(np.concatenate([r[0] for r in res], axis=0), want)
    assert all(r[1] == int(np.sum(want != want_prev)) for r in res)


def test_eikonal_validation():
    g = B.Grid(2, (64, 64)).decompose((64, 64))
    with pytest.raises(B.SweepError):
        g.eikonal_sweep(1, 0)                                   # no slowness yet
    with pytest.raises(B.SweepError):
        g.set_slowness(np.zeros((64, 64)), 0.1)                 # f must be > 0
    with pytest.raises(B.SweepError):
        g.set_slowness(np.ones((64, 64)), 0.0)                  # h must be > 0
    g3 = B.Grid(3, (8, 8, 8)).decompose((8, 8, 8))
    with pytest.raises(B.SweepError):
        g3.set_slowness(np.ones((8, 8, 8)), 0.1)                # 2D only
    g4 = B.Grid(2, (256, 128)).decompose((128, 64))
    g4.set_slowness(np.ones((128, 256)), 0.1)
    with pytest.raises(B.SweepError):
        g4.eikonal_sweep(1, 0)                                  # boxes larger than 64 x 64
