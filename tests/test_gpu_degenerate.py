"""Degenerate and boundary cases of the method through the C ABI, against the oracle: a single node,
boxes of one node (every node a box, so coupled sets everywhere: 2 x 2 pairs in 1D, 4-cycles in 2D,
8-cycles in 3D), boxes of two nodes, a singular coupled system (SW_ESINGULAR on both sides) and
invalid arguments (SW_EINVAL, never a silent fallback)."""
import numpy as np
import pytest

import oracle as O
from paper_1008_3699_b200 import binding as B, gen
from tests.gpu_helpers import make_grid, rand_faces

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,tile,var", [((1,), (1,), False), ((7,), (1,), True), ((6, 5), (1, 1), True),
                                        ((6, 6), (2, 3), False), ((4, 3, 2), (1, 1, 1), True),
                                        ((6, 6, 6), (2, 2, 2), True), ((2, 2, 2), (2, 2, 2), False)])
def test_tiny_boxes_match_oracle(n, tile, var):
    faces = rand_faces(n, 23) if var else None
    pb = O.tiled(n, tile, faces=faces, beta=0.05)
    g = make_grid(B, n, tile, faces, 0.05)
    x = gen.uniform_field(3, gen.STREAM_X0, pb.shape)
    b = gen.uniform_field(3, gen.STREAM_RHS, pb.shape)
    g.set_vector(B.X, x)
    g.set_vector(B.B, b)
    omega = [1.1]
    ph = 0
    for k in range(2 ** len(n) + 1):
        x = O.sweep(pb, omega, x, b, phase=k)
        ph = g.sor_sweep(omega, 1, ph)
        assert np.array_equal(g.get_vector(B.X), x), k
    g.check()
    # the preconditioners on the same boxes
    r = gen.uniform_field(4, gen.STREAM_TEST, pb.shape)
    g.set_vector(B.R, r)
    g.ssor_apply(1.0, g.ptr(B.R), g.ptr(B.Z), B.PAIR_SYMMETRIC)
    assert np.array_equal(g.get_vector(B.Z), O.ssor_apply(pb, 1.0, r, 0))
    g.ilu0_factor(0)
    g.ilu_apply(g.ptr(B.R), g.ptr(B.Z), B.PAIR_SYMMETRIC)
    assert np.array_equal(g.get_vector(B.Z), O.ilu_apply(pb, O.ilu0_factor(pb), r, 0))


def test_singular_coupled_pair_is_reported():
    # two one-node boxes; with tiny outer faces the coupled pair's determinant 1 - r1 r2 vanishes
    n, tile = (2,), (1,)
    faces = (np.array([1e-16, 1.0, 1e-16]),)
    pb = O.tiled(n, tile, faces=faces)
    b = np.ones(2)
    O.sweep(pb, [1.0], np.zeros(2), b, phase=0)          # phase 0: the shared face is an end face
    with pytest.raises(O.OracleError):
        O.sweep(pb, [1.0], np.zeros(2), b, phase=1)      # phase 1: both boxes start there
    g = make_grid(B, n, tile, faces)
    g.set_vector(B.B, b)
    g.sor_sweep([1.0], 1, 0)
    g.check()
    g.sor_sweep([1.0], 1, 1)
    with pytest.raises(B.SweepError) as e:
        g.check()
    assert e.value.code == B.SW_ESINGULAR


def test_invalid_arguments_are_rejected():
    with pytest.raises(B.SweepError):
        B.Grid(2, (100, 64), B.COEF_POISSON).decompose((64, 64))          # tile does not divide n
    g = make_grid(B, (64, 64), (64, 64))
    for w in ([0.0], [2.0], [-0.5], [1.0, 1.0, 1.0]):                     # omega outside (0, 2); 3 values in 2D
        with pytest.raises(B.SweepError):
            g.sor_sweep(w, 1, 0)
    with pytest.raises(B.SweepError):
        g.ilu_apply(g.ptr(B.R), g.ptr(B.Z), B.PAIR_SYMMETRIC)              # factor must come first
