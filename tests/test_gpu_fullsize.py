"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times (64 x 64 boxes
for configs 3 and 4, 512 x 8 x 4 for config 5, plus the 32 x 8 x 4 comparison line), on sampled
outputs the oracle computes one by one.

A box's part of a decomposed sweep depends only on the old values, b and faces within two layers
of the box (tile locality, SURVEY §8(c) C-SOR 2).  So the oracle sweeps a sub-grid of a few boxes
around a sampled box, cut out of the full-size inputs (starting at an even box index, so every
box keeps its direction bits, and running to the domain's own boundary where the box touches it),
and the sampled box of that sweep must equal the full-size GPU sweep bit for bit.  The PCG check
at full size is the property that holds at any size: the oracle's residual of the GPU solution."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_1008_3699_b200 import binding as B, gen

pytestmark = pytest.mark.gpu


def sub_range(bi, nb, T):
    """[lo, hi) node range of the sub-grid around box bi (even first box, clipped to the domain)."""
    b0 = bi - 1 if (bi - 1) % 2 == 0 else bi - 2
    b0 = max(b0, 0)
    b1 = min(bi + 1, nb - 1)
    return b0 * T, (b1 + 1) * T


def sampled_boxes(nb, rng, extra=3):
    dim = len(nb)
    boxes = {tuple([0] * dim), tuple(v - 1 for v in nb), tuple([0] + [v - 1 for v in nb[1:]])}
    edge = [v // 2 for v in nb]
    edge[0] = 0
    boxes.add(tuple(edge))
    while len(boxes) < 4 + extra:
        boxes.add(tuple(int(rng.integers(0, v)) for v in nb))
    return sorted(boxes)


def check_boxes(n, tile, x0, b, xnew, omega, phase, k_ring=None, scale=None, nsample=3, seed=0):
    dim = len(n)
    nb = [v // t for v, t in zip(n, tile)]
    rng = np.random.default_rng(seed)
    for box in sampled_boxes(nb, rng, nsample):
        rngs = [sub_range(bi, nbi, T) for bi, nbi, T in zip(box, nb, tile)]
        sl = tuple(slice(lo, hi) for lo, hi in reversed(rngs))             # numpy order (z, y, x)
        nsub = tuple(hi - lo for lo, hi in rngs)
        faces = None
        if k_ring is not None:
            slk = tuple(slice(lo, hi + 2) for lo, hi in reversed(rngs))
            faces = O.faces_from_k(nsub, np.ascontiguousarray(k_ring[slk]), scale)
        pb = O.tiled(nsub, tile, faces=faces)
        got_sub = O.sweep(pb, omega, np.ascontiguousarray(x0[sl]), np.ascontiguousarray(b[sl]), phase)
        # the sampled box inside the sub-grid and inside the full grid
        in_sub = tuple(slice(bi * T - lo, (bi + 1) * T - lo) for bi, T, (lo, hi) in reversed(list(zip(box, tile, rngs))))
        in_full = tuple(slice(bi * T, (bi + 1) * T) for bi, T in reversed(list(zip(box, tile))))
        assert np.array_equal(xnew[in_full], got_sub[in_sub]), f"box {box}"


def test_config4_full_size_sampled_boxes():
    n, tile = (16384, 16384), (64, 64)
    omega = [2.0 / (1.0 + np.sin(np.pi / (n[0] + 1)))]
    shape = tuple(reversed(n))
    x0 = gen.uniform_field(11, gen.STREAM_X0, shape)
    b = gen.uniform_field(0, gen.STREAM_RHS, shape) / float((n[0] + 1) ** 2)
    g = B.Grid(2, n, B.COEF_POISSON).decompose(tile)
    g.set_vector(B.X, x0)
    g.set_vector(B.B, b)
    g.sor_sweep(omega, 1, 3)
    torch.cuda.synchronize()
    xnew = g.get_vector(B.X)
    g.check()
    check_boxes(n, tile, x0, b, xnew, omega, 3)


def test_config3_full_size_sampled_boxes_and_pcg():
    n, tile = (4096, 4096), (64, 64)
    shape = tuple(reversed(n))
    k = gen.lognormal_k(0, tuple(v + 2 for v in shape), 1.0)
    x0 = gen.uniform_field(12, gen.STREAM_X0, shape)
    b = gen.uniform_field(0, gen.STREAM_RHS, shape) / float((n[0] + 1) ** 2)
    g = B.Grid(2, n, B.COEF_FACES).decompose(tile)
    g.set_coefficients_k(np.pad(k, [(1, 1), (0, 0)], constant_values=1.0), (1.0, 1.0))   # as bench.py
    g.set_vector(B.X, x0)
    g.set_vector(B.B, b)
    g.sor_sweep([1.0], 1, 1)
    torch.cuda.synchronize()
    check_boxes(n, tile, x0, b, g.get_vector(B.X), [1.0], 1, k, (1.0, 1.0))
    # ILU(0)-PCG at full size: the oracle's residual of the GPU solution
    it, rel, ok = g.pcg_solve(B.PC_ILU0, 1.0, B.PAIR_SYMMETRIC, 1e-8, 20000)
    assert ok and rel < 1e-8
    pb = O.tiled(n, tile, faces=O.faces_from_k(n, k, (1.0, 1.0)))
    assert O.relres(pb, g.get_vector(B.X), b) < 2e-8


@pytest.mark.parametrize("tile", [(512, 8, 4), (32, 8, 4)])
def test_config5_full_size_sampled_boxes(tile):
    n = (512, 512, 512)
    shape = tuple(reversed(n))
    k = gen.lognormal_k(0, tuple(v + 2 for v in shape), 0.5)
    x0 = gen.uniform_field(13, gen.STREAM_X0, shape)
    b = gen.uniform_field(0, gen.STREAM_RHS, shape) / float((n[0] + 1) ** 2)
    g = B.Grid(3, n, B.COEF_FACES).decompose(tile)
    g.set_coefficients_k(np.pad(k, [(1, 1), (0, 0), (0, 0)], constant_values=1.0), (1.0, 0.1, 0.01))   # as bench.py
    g.set_vector(B.X, x0)
    g.set_vector(B.B, b)
    g.sor_sweep([1.0], 1, 5)
    torch.cuda.synchronize()
    check_boxes(n, tile, x0, b, g.get_vector(B.X), [1.0], 5, k, (1.0, 0.1, 0.01), nsample=4)


def test_config5_full_size_pcg():
    """ILU(0)-PCG on config 5's grid with bench.py's boxes: the oracle's residual of the GPU solution."""
    n, tile = (512, 512, 512), (512, 8, 4)
    shape = tuple(reversed(n))
    k = gen.lognormal_k(0, tuple(v + 2 for v in shape), 0.5)
    kp = np.pad(k, [(1, 1), (0, 0), (0, 0)], constant_values=1.0)
    b = gen.uniform_field(0, gen.STREAM_RHS, shape) / float((n[0] + 1) ** 2)
    g = B.Grid(3, n, B.COEF_FACES).decompose(tile)
    g.set_coefficients_k(kp, (1.0, 0.1, 0.01))
    g.set_vector(B.B, b)
    it, rel, ok = g.pcg_solve(B.PC_ILU0, 1.0, B.PAIR_SYMMETRIC, 1e-8, 5000)
    assert ok and rel < 1e-8
    x = g.get_vector(B.X)
    del g
    pb = O.tiled(n, tile, faces=O.faces_from_k(n, k, (1.0, 0.1, 0.01)))
    assert O.relres(pb, x, b) < 2e-8
