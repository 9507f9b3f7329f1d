"""Pins for the nine-point oracle (DESIGN R-N3), -m "not gpu": one box
against the textbook frontal nine-point SOR loop; zero diagonals reduce it bitwise to the five-point
sweep; every node's sweep equation checked in numpy with the start-side rule written out; the fixed
point against the dense solve of the nine-point matrix assembled independently; the Mehrstellen
Laplacian reproduces harmonic polynomials exactly; the corner set is the dense 4 x 4."""
import numpy as np
import pytest

import oracle as O
from paper_1008_3699_b200 import gen

NB9 = [(-1, 0), (1, 0), (0, -1), (0, 1), (-1, -1), (1, -1), (-1, 1), (1, 1)]


def rand_faces(n, seed, lo=0.5, hi=2.0):
    return tuple(lo + (hi - lo) * gen.unit(seed, gen.STREAM_TEST + a, int(np.prod(O.face_shape(n, a)))).reshape(
        O.face_shape(n, a)) for a in range(len(n)))


def rand_diag(n, seed, lo=0.1, hi=0.8):
    sh = O.diag_shape(n)
    return tuple(lo + (hi - lo) * gen.unit(seed, gen.STREAM_TEST + 5 + k, int(np.prod(sh))).reshape(sh)
                 for k in range(2))


def coef(faces, diag, n, x, y, dx, dy):
    """c_pq of p = (x, y) and q = p + (dx, dy), straight from the array definitions."""
    F = faces
    if dy == 0:
        return F[0][y, x + (dx > 0)] if F is not None else 1.0
    if dx == 0:
        return F[1][y + (dy > 0), x] if F is not None else 1.0
    cx, cy = x + (dx > 0), y + (dy > 0)
    return diag[0][cy, cx] if dx == dy else diag[1][cy, cx]


def dense_A9(n, faces, diag, beta=0.0):
    n0, n1 = n
    N = n0 * n1
    A = np.zeros((N, N))
    for y in range(n1):
        for x in range(n0):
            p = x + n0 * y
            s = 0.0
            for dx, dy in NB9:
                c = coef(faces, diag, n, x, y, dx, dy)
                s += c
                qx, qy = x + dx, y + dy
                if 0 <= qx < n0 and 0 <= qy < n1:
                    A[p, qx + n0 * qy] = -c
            A[p, p] = s + beta
    return A


@pytest.mark.parametrize("n", [(7, 6), (5, 9)])
def test_one_box_is_textbook_frontal_sor(n):
    F, Dg = rand_faces(n, 1), rand_diag(n, 2)
    pb = O.tiled(n, n, faces=F, beta=0.1)
    x0 = gen.uniform_field(1, gen.STREAM_X0, pb.shape)
    b = gen.uniform_field(1, gen.STREAM_RHS, pb.shape)
    for c in range(4):
        for w in (1.0, 1.3):
            got = O.sweep9(pb, Dg, [w], x0, b, override=c)
            want = O.sor9_frontal(pb, Dg, w, x0, b, corner=c)
            assert np.max(np.abs(got - want)) <= 1e-13 * np.max(np.abs(want)), (c, w)


@pytest.mark.parametrize("n,tile", [((12, 12), (4, 4)), ((10, 9), (5, 3)), ((8, 8), (1, 1)), ((6, 8), (2, 2))])
def test_zero_diagonals_reduce_to_the_five_point_sweep(n, tile):
    F = rand_faces(n, 3)
    Z = tuple(np.zeros(O.diag_shape(n)) for _ in range(2))
    pb = O.tiled(n, tile, faces=F, beta=0.05)
    x0 = gen.uniform_field(2, gen.STREAM_X0, pb.shape)
    b = gen.uniform_field(2, gen.STREAM_RHS, pb.shape)
    for k in range(5):
        assert np.array_equal(O.sweep9(pb, Z, [1.2], x0, b, phase=k), O.sweep(pb, [1.2], x0, b, phase=k)), k


@pytest.mark.parametrize("n,tile,phase", [((12, 10), (4, 5), 0), ((12, 10), (4, 5), 3), ((9, 8), (3, 2), 1),
                                          ((8, 8), (2, 2), 2), ((6, 6), (1, 1), 0)])
def test_every_node_satisfies_its_nine_point_sweep_equation(n, tile, phase):
    """a_P / w u+_p - sum_{q implicit} c u+_q = a_P (1/w - 1) u_p + b_p + sum_{q explicit} c u_q at every
    node, with q implicit iff it lies on the start side of p's box along every axis where they differ
    (R-N3) and the box directions of R-4/R-5.  Catches a wrong classification of a diagonal, a wrong
    diagonal index, or a coupled set solved with an old partner value."""
    F, Dg = rand_faces(n, 4), rand_diag(n, 5)
    pb = O.tiled(n, tile, faces=F)
    x0 = gen.uniform_field(3, gen.STREAM_X0, pb.shape)
    b = gen.uniform_field(3, gen.STREAM_RHS, pb.shape)
    w = 1.15
    xn = O.sweep9(pb, Dg, [w], x0, b, phase=phase)
    cyc = [(1, 1), (0, 0), (0, 1), (1, 0)][phase % 4]
    n0, n1 = n
    worst = 0.0
    for y in range(n1):
        for x in range(n0):
            sx = cyc[0] ^ ((x // tile[0]) & 1)
            sy = cyc[1] ^ ((y // tile[1]) & 1)
            ap = sum(coef(F, Dg, n, x, y, dx, dy) for dx, dy in NB9)
            lhs = ap / w * xn[y, x]
            rhs = ap * (1 / w - 1) * x0[y, x] + b[y, x]
            for dx, dy in NB9:
                qx, qy = x + dx, y + dy
                if not (0 <= qx < n0 and 0 <= qy < n1):
                    continue
                start_x = dx == 0 or dx == (1 if sx else -1)
                start_y = dy == 0 or dy == (1 if sy else -1)
                c = coef(F, Dg, n, x, y, dx, dy)
                if start_x and start_y:
                    lhs -= c * xn[qy, qx]
                else:
                    rhs += c * x0[qy, qx]
            worst = max(worst, abs(lhs - rhs))
    assert worst <= 1e-12, worst


def test_fixed_point_is_the_nine_point_solution():
    """Sweeps converge to A9^-1 b with A9 assembled here from the coefficient definitions."""
    n, tile = (12, 10), (4, 5)
    F, Dg = rand_faces(n, 6), rand_diag(n, 7)
    pb = O.tiled(n, tile, faces=F, beta=0.3)
    b = gen.uniform_field(4, gen.STREAM_RHS, pb.shape)
    x = np.zeros(pb.shape)
    for k in range(400):
        x = O.sweep9(pb, Dg, [1.0], x, b, phase=k)
    A = dense_A9(n, F, Dg, 0.3)
    want = np.linalg.solve(A, b.ravel())
    assert np.max(np.abs(x.ravel() - want)) <= 1e-11 * np.max(np.abs(want))


def test_mehrstellen_reproduces_harmonic_polynomials():
    """The nine-point Mehrstellen Laplacian (axis 4, diagonal 1, a_P = 20) is exact for harmonic
    polynomials such as x y and x^2 - y^2: with their boundary values folded into b the converged
    decomposed sweep returns them at the nodes."""
    n, tile = (10, 10), (5, 5)
    n0, n1 = n
    F = tuple(np.full(O.face_shape(n, a), 4.0) for a in range(2))
    Dg = tuple(np.ones(O.diag_shape(n)) for _ in range(2))
    pb = O.tiled(n, tile, faces=F)
    h = 1.0 / (n0 + 1)
    for fun in (lambda X, Y: X * Y, lambda X, Y: X * X - Y * Y, lambda X, Y: 3 * X - 2 * Y + 1):
        b = np.zeros(pb.shape)
        for y in range(n1):
            for x in range(n0):
                for dx, dy in NB9:
                    qx, qy = x + dx, y + dy
                    if not (0 <= qx < n0 and 0 <= qy < n1):
                        b[y, x] += coef(F, Dg, n, x, y, dx, dy) * fun((qx + 1) * h, (qy + 1) * h)
        u = np.zeros(pb.shape)
        for k in range(600):
            u = O.sweep9(pb, Dg, [1.0], u, b, phase=k)
        Y, X = np.mgrid[1:n1 + 1, 1:n0 + 1] * h
        assert np.max(np.abs(u - fun(X, Y))) <= 1e-11


def test_corner_set_is_dense_four_by_four():
    """On 2 x 2 boxes at phase 0 (all four boxes start at the centre) the centre 2 x 2 nodes form one
    coupled set whose matrix has all 12 off-diagonal couplings (the five-point sweep: 8): the
    iteration matrix of one sweep restricted to them is dense; away from it only pairs couple."""
    n, tile = (6, 6), (3, 3)
    Dg = rand_diag(n, 8)
    pb = O.tiled(n, tile)
    N = pb.size
    z = np.zeros(pb.shape)
    # response of the four centre nodes to a unit right-hand side at each of them
    centre = [(2, 2), (2, 3), (3, 2), (3, 3)]        # (y, x)
    resp9 = np.zeros((4, 4))
    resp5 = np.zeros((4, 4))
    Z = tuple(np.zeros(O.diag_shape(n)) for _ in range(2))
    for j, (y, x) in enumerate(centre):
        e = np.zeros(pb.shape)
        e[y, x] = 1.0
        u9 = O.sweep9(pb, Dg, [1.0], z, e, phase=0)
        u5 = O.sweep9(pb, Z, [1.0], z, e, phase=0)
        for i, (yy, xx) in enumerate(centre):
            resp9[i, j] = u9[yy, xx]
            resp5[i, j] = u5[yy, xx]
    assert np.all(np.abs(resp9) > 0)                  # every centre node depends on every other
    assert N == 36
    # the five-point set is a 4-cycle: still all positive (inverse of an irreducible M-matrix)
    assert np.all(np.abs(resp5) > 0) and not np.allclose(resp9, resp5)
