"""Pins for the eikonal oracle (DESIGN R-E1..R-E3), -m "not gpu": the decomposed
fast-sweeping pass against the textbook fast-sweeping loop (one box), closed forms (1D first-arrival
sums, 2D axis lines and the first diagonal node), the Godunov equation at the fixed point written
out independently in numpy, monotonicity, and first-order convergence to the exact distance."""
import numpy as np
import pytest

import oracle as O
from paper_1008_3699_b200 import gen

INF = np.inf


def slowness(shape, seed, lo=0.5, hi=2.0):
    return lo + (hi - lo) * gen.unit(seed, gen.STREAM_TEST, int(np.prod(shape))).reshape(shape)


def point_source(shape, idx):
    u = np.full(shape, INF)
    u[idx] = 0.0
    return u


def converge(step, u, limit=500):
    for it in range(limit):
        un = step(u, it)
        if np.array_equal(un, u):
            return un, it
        u = un
    raise AssertionError("no convergence")


def godunov_np(a, b, fh):
    """The Godunov solution written out in numpy (same formula as R-E1, vectorised)."""
    m = np.minimum(a, b)
    with np.errstate(invalid="ignore"):
        d = a - b
        two = 0.5 * ((a + b) + np.sqrt(np.maximum(2.0 * fh * fh - d * d, 0.0)))
    out = np.where(np.abs(d) >= fh, m + fh, two)
    return np.where(np.isinf(m), INF, out)


def neighbour_mins(u):
    pad = np.pad(u, 1, constant_values=INF)
    a = np.minimum(pad[1:-1, :-2], pad[1:-1, 2:])
    b = np.minimum(pad[:-2, 1:-1], pad[2:, 1:-1])
    return a, b


@pytest.mark.parametrize("n", [(13, 9), (8, 8), (30,)])
def test_one_box_is_classical_fast_sweeping(n):
    """With one box and a fixed corner the decomposed pass is the textbook in-place fast-sweeping
    loop from that corner, bit for bit (both the ordering and the update rule)."""
    pb = O.tiled(n, n)
    shape = pb.shape
    f = slowness(shape, 3)
    u = np.where(gen.unit(4, gen.STREAM_TEST, pb.size).reshape(shape) < 0.2, 0.0, INF)
    u[(0,) * len(shape)] = 0.0
    h = 1.0 / 16
    for c in range(2 ** len(n)):
        for _ in range(3):
            want = O.eik_classical(pb, c, f, h, u)
            got = O.eik_sweep(pb, f, h, u, override=c)
            assert np.array_equal(got, want), c
            u = want


def test_1d_first_arrival_sums():
    """1D: u_i = u_{i-1} + f_i h away from the source (exact first-arrival times)."""
    n = 40
    pb = O.tiled((n,), (8,))
    f = slowness((n,), 5)
    h = 0.1
    u, _ = converge(lambda v, k: O.eik_sweep(pb, f, h, v, phase=k), point_source((n,), 17))
    want = np.zeros(n)
    for i in range(18, n):
        want[i] = want[i - 1] + f[i] * h
    for i in range(16, -1, -1):
        want[i] = want[i + 1] + f[i] * h
    assert np.array_equal(u, want)


def test_2d_constant_speed_closed_forms():
    """f = 1, one source: u = |offset| h along the source's row and column; the first diagonal
    node has a = b = h, so u = h (1 + 1/sqrt(2)) (the Godunov two-term solution)."""
    n, tile = (24, 20), (6, 5)
    pb = O.tiled(n, tile)
    f = np.ones(pb.shape)
    h = 0.05
    s = (9, 11)                                      # (y, x)
    u, _ = converge(lambda v, k: O.eik_sweep(pb, f, h, v, phase=k), point_source(pb.shape, s))
    ys, xs = s
    for x in range(n[0]):
        assert abs(u[ys, x] - abs(x - xs) * h) <= 1e-13
    for y in range(n[1]):
        assert abs(u[y, xs] - abs(y - ys) * h) <= 1e-13
    for dy, dx in ((1, 1), (-1, 1), (1, -1), (-1, -1)):
        assert abs(u[ys + dy, xs + dx] - h * (1 + 1 / np.sqrt(2))) <= 1e-15


@pytest.mark.parametrize("n,tile", [((40, 36), (8, 9)), ((32, 32), (4, 4)), ((17, 23), (17, 23))])
def test_decomposed_converges_to_the_classical_solution(n, tile):
    """The discrete viscosity solution is unique: the decomposed sweeps converge to the same grid
    function as classical fast sweeping (to rounding), which satisfies the Godunov equation
    (u - a)+^2 + (u - b)+^2 = (f h)^2 at every non-source node (checked in numpy); every pass is
    monotone (u never increases)."""
    pb = O.tiled(n, tile)
    one = O.tiled(n, n)
    f = slowness(pb.shape, 7)
    h = 1.0 / max(n)
    u0 = point_source(pb.shape, (3, 5))
    u0[pb.shape[0] - 2, pb.shape[1] - 4] = 0.0

    def dec(v, k):
        w = O.eik_sweep(pb, f, h, v, phase=k)
        assert np.all(w <= v)
        return w
    ud, itd = converge(dec, u0)
    uc, itc = converge(lambda v, k: O.eik_classical(one, [0, 1, 3, 2][k % 4], f, h, v), u0)
    assert np.max(np.abs(ud - uc)) <= 1e-13 * np.max(uc)
    a, b = neighbour_mins(ud)
    fh = f * h
    src = ud == 0.0
    res = np.maximum(ud - a, 0.0) ** 2 + np.maximum(ud - b, 0.0) ** 2 - fh * fh
    assert np.max(np.abs(res[~src])) <= 1e-12 * np.max(fh * fh)
    assert np.array_equal(godunov_np(a, b, fh)[~src], ud[~src]) or \
        np.max(np.abs(godunov_np(a, b, fh)[~src] - ud[~src])) <= 1e-14 * np.max(ud)


def test_converges_to_the_distance_function():
    """f = 1: the first-order Godunov scheme converges to the Euclidean distance; halving h cuts
    the max error (of order h log(1/h)) by more than 1.5x."""
    errs = []
    for m in (16, 32, 64):
        n = (m + 1, m + 1)
        pb = O.tiled(n, n)
        h = 1.0 / m
        c = m // 2
        u, _ = converge(lambda v, k: O.eik_sweep(pb, np.ones(pb.shape), h, v, phase=k), point_source(pb.shape, (c, c)))
        yy, xx = np.mgrid[0:m + 1, 0:m + 1]
        exact = h * np.sqrt((yy - c) ** 2 + (xx - c) ** 2)
        errs.append(np.max(np.abs(u - exact)))
    assert errs[0] / errs[1] > 1.5 and errs[1] / errs[2] > 1.5, errs


@pytest.mark.parametrize("n,tile,phase", [((12, 10), (4, 5), 0), ((12, 10), (4, 5), 1), ((9, 8), (3, 2), 2),
                                          ((9, 8), (3, 2), 3), ((8, 8), (1, 1), 0)])
def test_every_node_satisfies_its_sweep_equation(n, tile, phase):
    """One decomposed pass, checked node by node in numpy: u+_p = min(u_p, Godunov(a, b)) with the
    NEW values of the neighbours on the start side of p's box and OLD values elsewhere (R-E2).  At
    the coupled sets (start-start faces) both members use each other's new value, so a set solved
    with an old partner value, or in the wrong order, fails here (R-E3).  The box directions come
    from the paper's rule s_a = c_a(k) XOR (r_a mod 2), c = [NE, SW, NW, SE] (R-4, R-5)."""
    pb = O.tiled(n, tile)
    ny, nx = pb.shape
    f = slowness(pb.shape, 9)
    h = 0.1
    u0 = np.where(gen.unit(10, gen.STREAM_TEST, pb.size).reshape(pb.shape) < 0.1, 0.0, INF)
    rng = gen.unit(11, gen.STREAM_TEST, pb.size).reshape(pb.shape)
    u0 = np.where(np.isinf(u0) & (rng < 0.5), 3.0 * rng, u0)           # finite old values too
    un = O.eik_sweep(pb, f, h, u0, phase=phase)
    cyc = [(1, 1), (0, 0), (0, 1), (1, 0)][phase % 4]                   # (sx, sy) of c(k)
    for y in range(ny):
        for x in range(nx):
            sx = cyc[0] ^ ((x // tile[0]) & 1)
            sy = cyc[1] ^ ((y // tile[1]) & 1)

            def val(qy, qx, implicit):
                if not (0 <= qx < nx and 0 <= qy < ny):
                    return INF
                return un[qy, qx] if implicit else u0[qy, qx]
            a = min(val(y, x - 1, sx == 0), val(y, x + 1, sx == 1))
            b = min(val(y - 1, x, sy == 0), val(y + 1, x, sy == 1))
            want = min(u0[y, x], godunov_np(np.array(a), np.array(b), np.array(f[y, x] * h)).item())
            assert un[y, x] == want or abs(un[y, x] - want) <= 1e-15 * max(abs(want), 1.0), (y, x)
