"""m-step preconditioners ("a few iterations of SOR ... during
each step of preconditioning"): z_1 = P^-1 r, z_{j+1} = z_j + P^-1 (r - A z_j) through the C ABI
(sw_set_precond_steps) against the same composition of oracle calls, and inside PCG."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_1008_3699_b200 import binding as B, gen
from tests.gpu_helpers import make_grid, rand_faces, rel_maxdiff

pytestmark = pytest.mark.gpu


def oracle_msteps(pb, r, m, pc, omega, pairing, invd=None, theta=0.5):
    def P(v):
        return O.ilu_apply(pb, invd, v, pairing) if pc == B.PC_ILU0 else O.ssor_apply(pb, omega, v, pairing)
    z = P(r)
    for _ in range(m - 1):
        z = z + P(r - theta * O.apply_A(pb, z))
    return z


CASES = [((128, 128), (64, 64), True), ((192, 128), (64, 64), False), ((32, 16, 16), (16, 8, 4), True),
         ((64, 32, 16), (32, 8, 4), True)]


@pytest.mark.parametrize("n,tile,var", CASES)
@pytest.mark.parametrize("pc", [B.PC_SSOR, B.PC_ILU0])
@pytest.mark.parametrize("m,theta", [(2, 0.5), (3, 1.0), (3, 0.7)])
def test_msteps_apply_matches_oracle(n, tile, var, pc, m, theta):
    faces = rand_faces(n, 13) if var else None
    pb = O.tiled(n, tile, faces=faces)
    r = gen.uniform_field(4, gen.STREAM_TEST, pb.shape)
    omega, pairing = 1.1, B.PAIR_SYMMETRIC
    g = make_grid(B, n, tile, faces).set_precond_steps(m, theta)
    invd = None
    if pc == B.PC_ILU0:
        g.ilu0_factor(0)
        invd = O.ilu0_factor(pb)
    g.set_vector(B.R, r)
    if pc == B.PC_ILU0:
        g.ilu_apply(g.ptr(B.R), g.ptr(B.Z), pairing)
    else:
        g.ssor_apply(omega, g.ptr(B.R), g.ptr(B.Z), pairing)
    torch.cuda.synchronize()
    got = g.get_vector(B.Z)
    want = oracle_msteps(pb, r, m, pc, omega, pairing, invd, theta)
    assert rel_maxdiff(got, want) <= 1e-12


@pytest.mark.parametrize("pc", [B.PC_SSOR, B.PC_ILU0])
def test_msteps_pcg_converges_in_fewer_iterations(pc):
    """theta = 1/2 keeps every m positive definite (lambda_max(P^-1 A) = 2 for the decomposed
    preconditioners) and the iteration count falls with m."""
    n, tile = (256, 256), (64, 64)
    pb = O.tiled(n, tile)
    b = gen.uniform_field(0, gen.STREAM_RHS, pb.shape) / float((n[0] + 1) ** 2)
    its = []
    for m in (1, 2, 3):
        g = make_grid(B, n, tile).set_precond_steps(m, 0.5)
        g.set_vector(B.B, b)
        it, rel, ok = g.pcg_solve(pc, 1.0, B.PAIR_SYMMETRIC, 1e-8, 5000)
        assert ok
        assert O.relres(pb, g.get_vector(B.X), b) < 2e-8
        its.append(it)
    assert its[0] > its[1] > its[2]


def test_precond_steps_validation():
    g = make_grid(B, (64, 64), (64, 64))
    with pytest.raises(B.SweepError):
        g.set_precond_steps(0)
    with pytest.raises(B.SweepError):
        g.set_precond_steps(65)
    with pytest.raises(B.SweepError):
        g.set_precond_steps(2, 1.5)
