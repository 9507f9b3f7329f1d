"""Geometric multigrid with the decomposed sweep as smoother: one V-cycle
through the C ABI (sw_mg_setup / sw_mg_apply) against the same V-cycle composed from oracle calls
(piecewise-constant aggregation, Galerkin face sums, m-step SGS smoothing, DESIGN R-17/R-19), and
MG-preconditioned CG."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_1008_3699_b200 import binding as B, gen
from tests.gpu_helpers import make_grid, rand_faces, rel_maxdiff
from tests.mg_compose import build_levels, vcycle

pytestmark = pytest.mark.gpu


CASES = [((256, 256), (64, 64), False, 0.0, 3, 0), ((128, 128), (64, 64), True, 0.0, 4, 0),
         ((64, 32, 32), (32, 8, 4), True, 0.0, 3, 0), ((32, 32, 32), (16, 8, 4), False, 0.1, 3, 0),
         ((64, 32, 16), (32, 8, 4), True, 0.0, 3, 3), ((128, 64), (64, 64), True, 0.05, 3, 1),
         ((32, 32, 16), (16, 8, 4), True, 0.0, 3, 5)]


@pytest.mark.parametrize("n,tile,var,beta,levels,axes", CASES)
@pytest.mark.parametrize("nu,theta,sc", [(1, 0.5, 1.0), (2, 0.6, 1.7)])
def test_vcycle_matches_oracle(n, tile, var, beta, levels, axes, nu, theta, sc):
    faces = rand_faces(n, 17) if var else None
    mask = axes or (1 << len(n)) - 1
    pbs = build_levels(n, tile, faces, beta, levels, mask)
    r = gen.uniform_field(8, gen.STREAM_TEST, pbs[0].shape)
    g = make_grid(B, n, tile, faces, beta).mg_setup(levels, nu, theta, 6, sc, axes)
    g.set_vector(B.R, r)
    g.mg_apply(g.ptr(B.R), g.ptr(B.Z))
    torch.cuda.synchronize()
    g.check()
    want = vcycle(pbs, 0, r, nu, theta, 6, sc, mask)
    assert rel_maxdiff(g.get_vector(B.Z), want) <= 1e-12


@pytest.mark.parametrize("n,tile,var,beta,levels,axes", [((256, 256), (64, 64), True, 0.0, 4, 0),
                                                         ((64, 32, 16), (32, 8, 4), True, 0.0, 4, 3),
                                                         ((32, 32, 32), (16, 8, 4), False, 0.1, 3, 0)])
def test_wcycle_matches_oracle(n, tile, var, beta, levels, axes):
    """gamma = 2 (sw_mg_set_cycle): every level above the coarsest corrects twice."""
    faces = rand_faces(n, 23) if var else None
    mask = axes or (1 << len(n)) - 1
    pbs = build_levels(n, tile, faces, beta, levels, mask)
    r = gen.uniform_field(9, gen.STREAM_TEST, pbs[0].shape)
    g = make_grid(B, n, tile, faces, beta).mg_setup(levels, 1, 0.5, 4, 1.2, axes).mg_set_cycle(2)
    g.set_vector(B.R, r)
    g.mg_apply(g.ptr(B.R), g.ptr(B.Z))
    torch.cuda.synchronize()
    g.check()
    want = vcycle(pbs, 0, r, 1, 0.5, 4, 1.2, mask, gamma=2)
    assert rel_maxdiff(g.get_vector(B.Z), want) <= 1e-12
    g.mg_set_cycle(1)                                   # back to the V-cycle
    g.mg_apply(g.ptr(B.R), g.ptr(B.Z))
    torch.cuda.synchronize()
    assert rel_maxdiff(g.get_vector(B.Z), vcycle(pbs, 0, r, 1, 0.5, 4, 1.2, mask)) <= 1e-12
    with pytest.raises(B.SweepError):
        g.mg_set_cycle(3)


@pytest.mark.parametrize("n,tile,var,levels", [((256, 256), (64, 64), True, 4), ((64, 64, 64), (32, 8, 4), True, 3)])
def test_mg_pcg_converges_in_few_iterations(n, tile, var, levels):
    faces = rand_faces(n, 19) if var else None
    pb = O.tiled(n, tile, faces=faces)
    b = gen.uniform_field(0, gen.STREAM_RHS, pb.shape) / float((n[0] + 1) ** 2)
    g = make_grid(B, n, tile, faces)
    g.set_vector(B.B, b)
    it_ilu, _, ok = g.pcg_solve(B.PC_ILU0, 1.0, B.PAIR_SYMMETRIC, 1e-8, 5000)
    assert ok
    g.mg_setup(levels, 1, 0.5, 16)
    it_mg, rel, ok = g.pcg_solve(B.PC_MG, 1.0, B.PAIR_SYMMETRIC, 1e-8, 5000)
    assert ok and it_mg < it_ilu / 2, (it_mg, it_ilu)
    assert O.relres(pb, g.get_vector(B.X), b) < 2e-8


def test_mg_setup_validation():
    g = make_grid(B, (192, 192), (64, 64))
    with pytest.raises(B.SweepError):
        g.mg_setup(1)
    with pytest.raises(B.SweepError):
        g.mg_setup(8)            # 192 -> 96 -> 48 -> 24 -> 12 -> 6 -> 3, then an odd count
    g2 = make_grid(B, (192, 192), (64, 64))
    with pytest.raises(B.SweepError):
        g2.mg_setup(3, 1, 1.5)
    with pytest.raises(B.SweepError):
        make_grid(B, (192, 192), (64, 64)).pcg_solve(B.PC_MG)


@pytest.mark.parametrize("law", ["poisson", "lognormal"])
def test_decomposed_smoother_loses_no_convergence(law):
    """The paper's claim that parallelising the sweep costs no convergence rate (PAPER:378-380
    "good smoothing properties", 2585-2588) measured where it matters most: the
    MG-PCG iteration count with the decomposed sweep as smoother on 64^2 / 32^2 / 16^2 boxes stays
    within 25 % of the same V-cycle with one box per level (the sequential sweep)."""
    n = (256, 256)
    b = gen.uniform_field(0, gen.STREAM_RHS, tuple(reversed(n))) / float((n[0] + 1) ** 2)
    faces = None
    if law == "lognormal":
        ring = tuple(v + 2 for v in reversed(n))
        faces = O.faces_from_k(n, gen.lognormal_k(0, ring, 1.0))
    its = {}
    for tile in [(256, 256), (64, 64), (32, 32), (16, 16)]:
        g = make_grid(B, n, tile, faces).mg_setup(4, 1, 0.5, 16, 1.2)
        g.set_vector(B.B, b)
        it, rel, ok = g.pcg_solve(B.PC_MG, 1.0, B.PAIR_SYMMETRIC, 1e-8, 5000)
        assert ok
        its[tile[0]] = it
    for t in (64, 32, 16):
        assert its[t] <= 1.25 * its[256], its
