"""Multi-rank data path on one GPU: the grid is split into slabs of whole tile rows (planes in
3D), each slab is its own library grid (rank r of R), and ghost layers move between them with
the same halo plan the NCCL transport uses (parallel.exchange_ghosts_local).  The decomposed
sweep and the preconditioner solves read only old values / redundantly recomputed partners
across box faces, so the slab results must equal the single-grid results bit for bit
(SURVEY §8(e)); the slab PCG sums rank partials in another order, so its iteration count may
differ by one."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_1008_3699_b200 import binding as B, gen, parallel
from tests.gpu_helpers import make_grid, rand_faces

pytestmark = pytest.mark.gpu


def slab_faces(faces, n, off, n_loc):
    """Slab-extended face arrays for sw_set_faces (2 extra layers per side of the slab axis)."""
    dim = len(n)
    out = []
    for a, f in enumerate(faces):
        f = np.asarray(f)
        ext = n_loc + 4 + (1 if a == dim - 1 else 0)
        shape = list(f.shape)
        shape[0] = ext
        e = np.zeros(shape)
        for j in range(ext):
            gj = off - 2 + j
            if 0 <= gj < f.shape[0]:
                e[j] = f[gj]
        out.append(e)
    return out


def make_slabs(n, tile, nranks, faces=None, beta=0.0):
    kind = B.COEF_POISSON if faces is None else B.COEF_FACES
    grids = []
    for r in range(nranks):
        g = B.Grid(len(n), n, kind, beta).decompose(tile, r, nranks)
        if faces is not None:
            g.set_faces_slab(slab_faces(faces, n, g.slab_offset, g.n_local[-1]))
        grids.append(g)
    return grids


def scatter(grids, which, full):
    for g in grids:
        sl = full[g.slab_offset:g.slab_offset + g.n_local[-1]]
        g.set_vector(which, np.ascontiguousarray(sl))


def gather(grids, which):
    return np.concatenate([g.get_vector(which) for g in grids], axis=0)


SWEEP_CASES = [((256, 256), (64, 64), 2, False), ((256, 256), (64, 64), 4, True), ((128, 192), (32, 32), 3, True),
               ((64, 32, 16), (32, 8, 4), 2, True), ((64, 16, 16), (32, 8, 4), 4, False)]


@pytest.mark.parametrize("n,tile,nranks,var", SWEEP_CASES)
def test_sweep_over_slabs_is_bitwise_single_grid(n, tile, nranks, var):
    faces = rand_faces(n, 7) if var else None
    pb = O.tiled(n, tile, faces=faces)
    x0 = gen.uniform_field(3, gen.STREAM_X0, pb.shape)
    b = gen.uniform_field(3, gen.STREAM_RHS, pb.shape)
    w = [1.3] if var else [1.9]
    one = make_grid(B, n, tile, faces)
    one.set_vector(B.X, x0)
    one.set_vector(B.B, b)
    sl = make_slabs(n, tile, nranks, faces)
    scatter(sl, B.X, x0)
    scatter(sl, B.B, b)
    parallel.exchange_ghosts_local([g.view(B.B) for g in sl], [g.n_local[-1] for g in sl], 2)
    nsw = 2 ** len(n) + 1
    one.sor_sweep(w, nsw, 0)
    for k in range(nsw):
        parallel.exchange_ghosts_local([g.view(B.X) for g in sl], [g.n_local[-1] for g in sl], 2)
        for g in sl:
            g.sor_sweep(w, 1, k)
    x = one.get_vector(B.X)
    assert np.isfinite(x).all()
    assert np.array_equal(gather(sl, B.X), x)


PC_CASES = [((256, 256), (64, 64), 2, True, B.PC_ILU0), ((256, 192), (64, 64), 3, False, B.PC_SSOR),
            ((96, 64), (32, 16), 2, True, B.PC_ILU0), ((32, 16, 16), (16, 8, 4), 2, True, B.PC_ILU0),
            ((32, 16, 16), (16, 8, 4), 4, False, B.PC_SSOR)]


@pytest.mark.parametrize("n,tile,nranks,var,pc", PC_CASES)
@pytest.mark.parametrize("pairing", [B.PAIR_SYMMETRIC, B.PAIR_PAPER])
def test_staged_preconditioner_over_slabs_is_bitwise_single_grid(n, tile, nranks, var, pc, pairing):
    faces = rand_faces(n, 11) if var else None
    pb = O.tiled(n, tile, faces=faces)
    r = gen.uniform_field(6, gen.STREAM_TEST, pb.shape)
    omega = 1.2
    one = make_grid(B, n, tile, faces)
    sl = make_slabs(n, tile, nranks, faces)
    if pc == B.PC_ILU0:
        one.ilu0_factor(0)
        for g in sl:
            g.ilu0_factor(0)
        parallel.exchange_ghosts_local([g.view(B.INVD) for g in sl], [g.n_local[-1] for g in sl], 1)
    one.set_vector(B.R, r)
    if pc == B.PC_ILU0:
        one.ilu_apply(one.ptr(B.R), one.ptr(B.Z), pairing)
    else:
        one.ssor_apply(omega, one.ptr(B.R), one.ptr(B.Z), pairing)
    scatter(sl, B.R, r)
    comm = parallel.LocalComm(sl)
    V = lambda w: [g.view(w) for g in sl]  # noqa: E731
    comm.exchange(V(B.R), 1)
    for st in range(sl[0].precond_stages(pairing)):
        if st == 1 and pairing == B.PAIR_PAPER:
            comm.exchange(V(B.Y), 1)
        if st >= 2:
            comm.exchange(V(B.Y), 1)
            comm.exchange(V(B.Z), 2)
        for g in sl:
            g.precond_apply_stage(pc, st, g.ptr(B.R), g.ptr(B.Z), omega, pairing)
    torch.cuda.synchronize()
    assert np.array_equal(gather(sl, B.Z), one.get_vector(B.Z))


@pytest.mark.parametrize("n,tile,nranks,var,pc", [((256, 256), (64, 64), 4, True, B.PC_ILU0),
                                                  ((192, 128), (64, 64), 2, False, B.PC_SSOR),
                                                  ((32, 16, 16), (16, 8, 4), 2, True, B.PC_ILU0),
                                                  ((128, 128), (32, 32), 2, True, B.PC_NONE)])
def test_pcg_over_slabs_matches_single_grid(n, tile, nranks, var, pc):
    faces = None
    if var:
        ring = tuple(v + 2 for v in reversed(n))
        faces = O.faces_from_k(n, gen.lognormal_k(0, ring, 1.0))
    pb = O.tiled(n, tile, faces=faces)
    b = gen.uniform_field(0, gen.STREAM_RHS, pb.shape) / float((n[0] + 1) ** 2)
    one = make_grid(B, n, tile, faces)
    one.set_vector(B.B, b)
    it1, rel1, ok1 = one.pcg_solve(pc, 1.0, 0, 1e-8, 5000)
    sl = make_slabs(n, tile, nranks, faces)
    scatter(sl, B.B, b)
    it, rel, ok = parallel.pcg_slabs(parallel.LocalComm(sl), pc, 1.0, 0, 1e-8, 5000)
    assert ok and ok1
    assert abs(it - it1) <= 1, (it, it1)
    x = gather(sl, B.X)
    assert O.relres(pb, x, b) < 2e-8


@pytest.mark.parametrize("n,tile,nranks,var,pc", [((256, 256), (64, 64), 2, True, B.PC_SSOR),
                                                  ((32, 16, 16), (16, 8, 4), 2, True, B.PC_ILU0)])
def test_msteps_pcg_over_slabs_matches_single_grid(n, tile, nranks, var, pc):
    """m-step preconditioning over slabs (staged solves + sw_apply_A + sw_axpby) reproduces the
    single-grid m-step PCG (sw_set_precond_steps)."""
    faces = None
    if var:
        ring = tuple(v + 2 for v in reversed(n))
        faces = O.faces_from_k(n, gen.lognormal_k(0, ring, 1.0))
    pb = O.tiled(n, tile, faces=faces)
    b = gen.uniform_field(0, gen.STREAM_RHS, pb.shape) / float((n[0] + 1) ** 2)
    one = make_grid(B, n, tile, faces).set_precond_steps(2, 0.5)
    one.set_vector(B.B, b)
    it1, rel1, ok1 = one.pcg_solve(pc, 1.0, 0, 1e-8, 5000)
    sl = make_slabs(n, tile, nranks, faces)
    scatter(sl, B.B, b)
    it, rel, ok = parallel.pcg_slabs(parallel.LocalComm(sl), pc, 1.0, 0, 1e-8, 5000, msteps=2, theta=0.5)
    assert ok and ok1
    assert abs(it - it1) <= 1, (it, it1)
    assert O.relres(pb, gather(sl, B.X), b) < 2e-8


@pytest.mark.parametrize("n,tile,nranks,var,pc", [((128, 128), (32, 32), 2, True, B.PC_ILU0),
                                                  ((32, 16, 16), (16, 8, 4), 2, True, B.PC_ILU0),
                                                  ((128, 128), (32, 32), 4, False, B.PC_SSOR)])
def test_flexible_pcg_over_slabs_matches_oracle(n, tile, nranks, var, pc):
    """The PAPER pairing over slabs: flexible (Polak-Ribiere) CG chosen automatically, iteration
    count within 1 of the single-grid sw_pcg_solve and of the oracle's flexible or_pcg."""
    faces = None
    if var:
        ring = tuple(v + 2 for v in reversed(n))
        faces = O.faces_from_k(n, gen.lognormal_k(0, ring, 1.0))
    pb = O.tiled(n, tile, faces=faces)
    b = gen.uniform_field(0, gen.STREAM_RHS, pb.shape) / float((n[0] + 1) ** 2)
    one = make_grid(B, n, tile, faces)
    one.set_vector(B.B, b)
    it1, rel1, ok1 = one.pcg_solve(pc, 1.0, B.PAIR_PAPER, 1e-8, 5000)
    _, ito, _, oko = O.pcg(pb, b, precond=pc, omega=1.0, pairing=1, flexible=True, rtol=1e-8, maxit=5000)
    sl = make_slabs(n, tile, nranks, faces)
    scatter(sl, B.B, b)
    it, rel, ok = parallel.pcg_slabs(parallel.LocalComm(sl), pc, 1.0, B.PAIR_PAPER, 1e-8, 5000)
    assert ok and ok1 and oko
    assert abs(it - it1) <= 1 and abs(it - ito) <= 1, (it, it1, ito)
    assert O.relres(pb, gather(sl, B.X), b) < 2e-8
