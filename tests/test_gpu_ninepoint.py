"""The nine-point decomposed SOR sweep through the C ABI (k_sweep9) against the
oracle's or_sweep9, bitwise, sweep after sweep: random symmetric coefficients and the Mehrstellen
Laplacian, several box shapes (coupled pairs, dense 4 x 4 corners, physical boundaries), per-direction
omega, slabs with the library's communicator; argument checks."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_1008_3699_b200 import binding as B, gen
from tests.gpu_helpers import rand_faces
from tests.slab_helpers import local_part, make_slab, run_threads

pytestmark = pytest.mark.gpu


def rand_diag(n, seed, lo=0.1, hi=0.8):
    sh = O.diag_shape(n)
    return tuple(lo + (hi - lo) * gen.unit(seed, gen.STREAM_TEST + 5 + k, int(np.prod(sh))).reshape(sh)
                 for k in range(2))


def mehrstellen(n):
    return (tuple(np.full(O.face_shape(n, a), 4.0) for a in range(2)), tuple(np.ones(O.diag_shape(n)) for _ in range(2)))


CASES = [((128, 96), (64, 32), "rand", 0.1, [1.3]), ((130, 66), (26, 22), "rand", 0.0, [0.7, 1.3, 1.1, 1.6]),
         ((64, 64), (64, 64), "rand", 0.0, [1.2]), ((40, 36), (8, 9), "mehr", 0.0, [1.5]),
         ((256, 192), (64, 64), "mehr", 0.0, [1.9]), ((24, 20), (1, 2), "rand", 0.2, [1.0]),
         ((33, 7), (3, 7), "poisson", 0.0, [1.4])]


@pytest.mark.parametrize("n,tile,law,beta,omega", CASES)
def test_nine_point_sweeps_match_oracle(n, tile, law, beta, omega):
    if law == "mehr":
        F, Dg = mehrstellen(n)
    elif law == "rand":
        F, Dg = rand_faces(n, 31), rand_diag(n, 32)
    else:
        F, Dg = None, rand_diag(n, 33)
    pb = O.tiled(n, tile, faces=F, beta=beta)
    x = gen.uniform_field(6, gen.STREAM_X0, pb.shape)
    b = gen.uniform_field(6, gen.STREAM_RHS, pb.shape)
    g = B.Grid(2, n, B.COEF_FACES if F is not None else B.COEF_POISSON, beta).decompose(tile)
    if F is not None:
        g.set_faces_global(F)
    g.set_diagonals(*Dg)
    g.set_vector(B.X, x)
    g.set_vector(B.B, b)
    ph = 0
    for k in range(5):
        x = O.sweep9(pb, Dg, omega, x, b, phase=k)
        ph = g.sor_sweep(omega, 1, ph)
        assert np.array_equal(g.get_vector(B.X), x), k
    g.check()


@pytest.mark.parametrize("n,tile,nranks", [((128, 256), (32, 32), 2), ((96, 192), (16, 16), 4), ((64, 96), (64, 8), 3)])
def test_nine_point_over_slabs_matches_oracle(n, tile, nranks):
    F, Dg = rand_faces(n, 34), rand_diag(n, 35)
    pb = O.tiled(n, tile, faces=F)
    x0 = gen.uniform_field(7, gen.STREAM_X0, pb.shape)
    b = gen.uniform_field(7, gen.STREAM_RHS, pb.shape)
    nsw = 6

    def rank_fn(r, comm):
        s = torch.cuda.Stream().cuda_stream
        g = make_slab(n, tile, r, nranks, F, 0.0, comm)
        g.set_diagonals(*Dg)
        g.set_vector(B.X, local_part(g, x0), stream=s)
        g.set_vector(B.B, local_part(g, b), stream=s)
        g.sor_sweep([1.25], nsw, 0, stream=s)
        return g.get_vector(B.X, stream=s)
    got = np.concatenate(run_threads(nranks, rank_fn), axis=0)
    x = x0
    for k in range(nsw):
        x = O.sweep9(pb, Dg, [1.25], x, b, phase=k)
    assert np.array_equal(got, x)


def test_nine_point_validation():
    n = (64, 64)
    g = B.Grid(2, n).decompose((64, 64))
    dd, da = rand_diag(n, 36)
    with pytest.raises(B.SweepError):
        g.set_diagonals(-dd, da)                             # coefficients >= 0
    g.set_diagonals(dd, da)
    with pytest.raises(B.SweepError):
        g.residual_norm()                                    # five-point only
    with pytest.raises(B.SweepError):
        g.pcg_solve(B.PC_ILU0)
    g3 = B.Grid(3, (8, 8, 8)).decompose((8, 8, 8))
    with pytest.raises(B.SweepError):
        g3.set_diagonals(np.ones((9, 9)), np.ones((9, 9)))   # 2D only
    g4 = B.Grid(2, (256, 128)).decompose((128, 64))
    g4.set_diagonals(np.ones((129, 257)), np.ones((129, 257)))
    with pytest.raises(B.SweepError):
        g4.sor_sweep([1.0], 1, 0)                            # boxes larger than 64 x 64
