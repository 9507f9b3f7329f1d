"""Multi-rank data path on one GPU, against the ORACLE.  The grid is split into slabs
of whole tile rows (planes in 3D), each slab its own library grid (rank r of R):

* staged (no communicator): the caller refreshes ghost layers between single sweeps / preconditioner
  stages with the halo plan the transports use (parallel.exchange_ghosts_local);
* in-library (a HOST communicator per rank, ranks as threads of this process sharing the GPU,
  parallel.ThreadHub): one sw_sor_sweep call of several sweeps with the boundary-rows-first /
  exchange-behind-the-interior schedule, sw_residual_norm, sw_ilu_apply / sw_ssor_apply (one and m
  steps) and sw_pcg_solve with device-side rank-ordered reductions.  (Processes instead of
  threads: tests/test_gpu_multiproc.py.)

Sweeps and preconditioner applications must equal the oracle bit for bit (boxes read only old
values / recompute coupled sets redundantly across slab faces); PCG iteration counts must be
within 1 of the oracle's and the solution's oracle residual < 2e-8."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_1008_3699_b200 import binding as B, gen, parallel
from tests.gpu_helpers import rand_faces, rel_maxdiff
from tests.slab_helpers import gather, local_part, make_slab, make_slabs, run_threads, scatter
from tests.test_gpu_msteps import oracle_msteps

pytestmark = pytest.mark.gpu


def oracle_sweeps(pb, w, x, b, nsw):
    for k in range(nsw):
        x = O.sweep(pb, w, x, b, phase=k)
    return x


SWEEP_CASES = [((256, 256), (64, 64), 2, False), ((256, 256), (64, 64), 4, True), ((128, 192), (32, 32), 3, True),
               ((64, 32, 16), (32, 8, 4), 2, True), ((64, 16, 16), (32, 8, 4), 4, False)]


@pytest.mark.parametrize("n,tile,nranks,var", SWEEP_CASES)
def test_staged_sweep_over_slabs_matches_oracle(n, tile, nranks, var):
    faces = rand_faces(n, 7) if var else None
    pb = O.tiled(n, tile, faces=faces)
    x0 = gen.uniform_field(3, gen.STREAM_X0, pb.shape)
    b = gen.uniform_field(3, gen.STREAM_RHS, pb.shape)
    w = [1.3] if var else [1.9]
    sl = make_slabs(n, tile, nranks, faces)
    scatter(sl, B.X, x0)
    scatter(sl, B.B, b)
    parallel.exchange_ghosts_local([g.view(B.B) for g in sl], [g.n_local[-1] for g in sl], 2)   # partners' b
    nsw = 2 ** len(n) + 1
    for k in range(nsw):
        parallel.exchange_ghosts_local([g.view(B.X) for g in sl], [g.n_local[-1] for g in sl], 2)
        for g in sl:
            g.sor_sweep(w, 1, k)
    assert np.array_equal(gather(sl, B.X), oracle_sweeps(pb, w, x0, b, nsw))


PC_CASES = [((256, 256), (64, 64), 2, True, B.PC_ILU0), ((256, 192), (64, 64), 3, False, B.PC_SSOR),
            ((96, 64), (32, 16), 2, True, B.PC_ILU0), ((32, 16, 16), (16, 8, 4), 2, True, B.PC_ILU0),
            ((32, 16, 16), (16, 8, 4), 4, False, B.PC_SSOR)]


def oracle_pc(pb, pc, r, omega, pairing):
    if pc == B.PC_ILU0:
        return O.ilu_apply(pb, O.ilu0_factor(pb), r, pairing)
    return O.ssor_apply(pb, omega, r, pairing)


@pytest.mark.parametrize("n,tile,nranks,var,pc", PC_CASES)
@pytest.mark.parametrize("pairing", [B.PAIR_SYMMETRIC, B.PAIR_PAPER])
def test_staged_preconditioner_over_slabs_matches_oracle(n, tile, nranks, var, pc, pairing):
    faces = rand_faces(n, 11) if var else None
    pb = O.tiled(n, tile, faces=faces)
    r = gen.uniform_field(6, gen.STREAM_TEST, pb.shape)
    omega = 1.2
    sl = make_slabs(n, tile, nranks, faces)
    if pc == B.PC_ILU0:
        for g in sl:
            g.ilu0_factor(0)
        parallel.exchange_ghosts_local([g.view(B.INVD) for g in sl], [g.n_local[-1] for g in sl], 1)
    scatter(sl, B.R, r)

    def exchange(w, width):
        parallel.exchange_ghosts_local([g.view(w) for g in sl], [g.n_local[-1] for g in sl], width)
    exchange(B.R, 1)
    for st in range(sl[0].precond_stages(pairing)):
        if st == 1 and pairing == B.PAIR_PAPER:
            exchange(B.Y, 1)
        if st >= 2:
            exchange(B.Y, 1)
            exchange(B.Z, 2)
        for g in sl:
            g.precond_apply_stage(pc, st, g.ptr(B.R), g.ptr(B.Z), omega, pairing)
    torch.cuda.synchronize()
    assert np.array_equal(gather(sl, B.Z), oracle_pc(pb, pc, r, omega, pairing))


# ------------------------------------------------------------------ in-library (communicator)
MR_SWEEP_CASES = [((256, 256), (64, 64), 2, False, 5),    # 2 tile rows per rank: no interior split
                  ((256, 512), (64, 64), 2, True, 5),     # 4 rows per rank: boundary rows + interior
                  ((192, 384), (64, 32), 3, True, 4),     # generic kernel, tile 32 along the slab axis
                  ((128, 64), (32, 4), 2, False, 6),      # tile 4: one boundary row per side
                  ((64, 32, 32), (32, 8, 4), 2, True, 9),  # 3D, z slabs of 4 boxes
                  ((64, 16, 48), (32, 8, 4), 3, False, 9),
                  ((240,), (10,), 3, True, 4),            # 1D: the slab axis is x
                  ((128, 96), (32, 1), 2, True, 3)]       # tile of 1 layer: 2 boundary rows per side


@pytest.mark.parametrize("n,tile,nranks,var,nsw", MR_SWEEP_CASES)
def test_multirank_sweeps_match_oracle(n, tile, nranks, var, nsw):
    """nsw sweeps in one sw_sor_sweep call per rank (exchanges inside the library) = the oracle's
    nsw sweeps bitwise; sw_residual_norm over ranks = the oracle's relative residual."""
    faces = rand_faces(n, 5) if var else None
    pb = O.tiled(n, tile, faces=faces, beta=0.05 if var else 0.0)
    x0 = gen.uniform_field(2, gen.STREAM_X0, pb.shape)
    b = gen.uniform_field(2, gen.STREAM_RHS, pb.shape)
    w = [1.2] if var else [1.7]

    def rank_fn(r, comm):
        s = torch.cuda.Stream()
        g = make_slab(n, tile, r, nranks, faces, pb.beta, comm)
        g.set_vector(B.X, local_part(g, x0), stream=s.cuda_stream)
        g.set_vector(B.B, local_part(g, b), stream=s.cuda_stream)
        ph = g.sor_sweep(w, nsw, 0, stream=s.cuda_stream)
        rel = g.residual_norm(stream=s.cuda_stream)
        g.check(stream=s.cuda_stream)
        return ph, g.get_vector(B.X, stream=s.cuda_stream), rel, g.launch_count()
    res = run_threads(nranks, rank_fn)
    want = oracle_sweeps(pb, w, x0, b, nsw)
    assert all(r[0] == nsw for r in res)
    assert np.array_equal(np.concatenate([r[1] for r in res], axis=0), want)
    rel_o = O.relres(pb, want, b)
    assert all(abs(r[2] - rel_o) <= 1e-12 * rel_o for r in res), ([r[2] for r in res], rel_o)


@pytest.mark.parametrize("n,tile,nranks,var,pc", PC_CASES + [((240,), (10,), 4, True, B.PC_ILU0)])
@pytest.mark.parametrize("pairing", [B.PAIR_SYMMETRIC, B.PAIR_PAPER])
def test_multirank_preconditioner_matches_oracle(n, tile, nranks, var, pc, pairing):
    faces = rand_faces(n, 11) if var else None
    pb = O.tiled(n, tile, faces=faces)
    r0 = gen.uniform_field(6, gen.STREAM_TEST, pb.shape)
    omega = 1.2

    def rank_fn(r, comm):
        s = torch.cuda.Stream().cuda_stream
        g = make_slab(n, tile, r, nranks, faces, 0.0, comm)
        g.set_vector(B.R, local_part(g, r0), stream=s)
        if pc == B.PC_ILU0:
            g.ilu0_factor(0, stream=s)
            g.ilu_apply(g.ptr(B.R), g.ptr(B.Z), pairing, stream=s)
        else:
            g.ssor_apply(omega, g.ptr(B.R), g.ptr(B.Z), pairing, stream=s)
        g.check(stream=s)
        return g.get_vector(B.Z, stream=s)
    got = np.concatenate(run_threads(nranks, rank_fn), axis=0)
    assert np.array_equal(got, oracle_pc(pb, pc, r0, omega, pairing))


@pytest.mark.parametrize("n,tile,nranks,pc", [((128, 256), (64, 64), 2, B.PC_SSOR), ((32, 16, 16), (16, 8, 4), 2, B.PC_ILU0)])
def test_multirank_msteps_matches_oracle(n, tile, nranks, pc):
    faces = rand_faces(n, 13)
    pb = O.tiled(n, tile, faces=faces)
    r0 = gen.uniform_field(4, gen.STREAM_TEST, pb.shape)

    def rank_fn(r, comm):
        s = torch.cuda.Stream().cuda_stream
        g = make_slab(n, tile, r, nranks, faces, 0.0, comm).set_precond_steps(3, 0.5)
        g.set_vector(B.R, local_part(g, r0), stream=s)
        if pc == B.PC_ILU0:
            g.ilu0_factor(0, stream=s)
            g.ilu_apply(g.ptr(B.R), g.ptr(B.Z), B.PAIR_SYMMETRIC, stream=s)
        else:
            g.ssor_apply(1.1, g.ptr(B.R), g.ptr(B.Z), B.PAIR_SYMMETRIC, stream=s)
        return g.get_vector(B.Z, stream=s)
    got = np.concatenate(run_threads(nranks, rank_fn), axis=0)
    invd = O.ilu0_factor(pb) if pc == B.PC_ILU0 else None
    want = oracle_msteps(pb, r0, 3, pc, 1.1, B.PAIR_SYMMETRIC, invd, 0.5)
    assert rel_maxdiff(got, want) <= 1e-12


MR_PCG_CASES = [((256, 256), (64, 64), 4, True, B.PC_ILU0, B.PAIR_SYMMETRIC),
                ((192, 128), (64, 64), 2, False, B.PC_SSOR, B.PAIR_SYMMETRIC),
                ((32, 16, 16), (16, 8, 4), 2, True, B.PC_ILU0, B.PAIR_SYMMETRIC),
                ((64, 32, 32), (32, 8, 4), 4, True, B.PC_SSOR, B.PAIR_SYMMETRIC),
                ((128, 128), (32, 32), 2, True, B.PC_NONE, B.PAIR_SYMMETRIC),
                ((128, 128), (32, 32), 2, True, B.PC_ILU0, B.PAIR_PAPER),      # flexible beta
                ((32, 16, 16), (16, 8, 4), 2, True, B.PC_SSOR, B.PAIR_PAPER)]


@pytest.mark.parametrize("n,tile,nranks,var,pc,pairing", MR_PCG_CASES)
def test_multirank_pcg_matches_oracle(n, tile, nranks, var, pc, pairing):
    faces = None
    if var:
        ring = tuple(v + 2 for v in reversed(n))
        faces = O.faces_from_k(n, gen.lognormal_k(0, ring, 1.0))
    pb = O.tiled(n, tile, faces=faces)
    b = gen.uniform_field(0, gen.STREAM_RHS, pb.shape) / float((n[0] + 1) ** 2)
    flexible = pairing == B.PAIR_PAPER

    def rank_fn(r, comm):
        s = torch.cuda.Stream().cuda_stream
        g = make_slab(n, tile, r, nranks, faces, 0.0, comm)
        g.set_vector(B.B, local_part(g, b), stream=s)
        it, rel, ok = g.pcg_solve(pc, 1.0, pairing, 1e-8, 5000, stream=s)
        return it, rel, ok, g.get_vector(B.X, stream=s)
    res = run_threads(nranks, rank_fn)
    _, ito, _, oko = O.pcg(pb, b, precond=pc, omega=1.0, pairing=pairing, flexible=flexible, rtol=1e-8, maxit=5000)
    its = {r[0] for r in res}
    assert len(its) == 1 and all(r[2] for r in res) and oko    # every rank took the same steps
    it = its.pop()
    assert abs(it - ito) <= 1, (it, ito)
    x = np.concatenate([r[3] for r in res], axis=0)
    assert O.relres(pb, x, b) < 2e-8


MG_CASES = [((128, 128), (16, 16), 2, True, 3, 0), ((64, 256), (16, 16), 4, False, 3, 0),
            ((32, 32, 32), (16, 8, 4), 2, True, 3, 0), ((64, 32, 16), (32, 8, 4), 2, True, 3, 3)]


@pytest.mark.parametrize("n,tile,nranks,var,levels,axes", MG_CASES)
def test_multirank_mg_vcycle_matches_oracle(n, tile, nranks, var, levels, axes):
    """The multigrid V-cycle over slabs (every level decomposed over the same ranks, ghost exchanges
    inside the library) against the oracle-side composition (tests/mg_compose.py), 1e-12."""
    from tests.mg_compose import build_levels, vcycle
    faces = rand_faces(n, 17) if var else None
    mask = axes or (1 << len(n)) - 1
    pbs = build_levels(n, tile, faces, 0.0, levels, mask)
    r0 = gen.uniform_field(8, gen.STREAM_TEST, pbs[0].shape)

    def rank_fn(r, comm):
        s = torch.cuda.Stream().cuda_stream
        g = make_slab(n, tile, r, nranks, faces, 0.0, comm).mg_setup(levels, 1, 0.5, 6, 1.3, axes)
        g.set_vector(B.R, local_part(g, r0), stream=s)
        g.mg_apply(g.ptr(B.R), g.ptr(B.Z), stream=s)
        g.check(stream=s)
        return g.get_vector(B.Z, stream=s)
    got = np.concatenate(run_threads(nranks, rank_fn), axis=0)
    want = vcycle(pbs, 0, r0, 1, 0.5, 6, 1.3, mask)
    assert rel_maxdiff(got, want) <= 1e-12


@pytest.mark.parametrize("n,tile,nranks,levels", [((256, 256), (16, 16), 2, 4), ((32, 32, 32), (16, 8, 4), 2, 3)])
def test_multirank_mg_pcg_matches_single_grid(n, tile, nranks, levels):
    """MG-preconditioned CG over slabs: iterations within 1 of the single-grid solve, solution's oracle
    residual < 2e-8."""
    ring = tuple(v + 2 for v in reversed(n))
    faces = O.faces_from_k(n, gen.lognormal_k(0, ring, 1.0))
    pb = O.tiled(n, tile, faces=faces)
    b = gen.uniform_field(0, gen.STREAM_RHS, pb.shape) / float((n[0] + 1) ** 2)
    one = B.Grid(len(n), n, B.COEF_FACES).decompose(tile)
    one.set_faces_global(faces)
    one.mg_setup(levels, 1, 0.5, 16)
    one.set_vector(B.B, b)
    it1, _, ok1 = one.pcg_solve(B.PC_MG, 1.0, B.PAIR_SYMMETRIC, 1e-8, 2000)

    def rank_fn(r, comm):
        s = torch.cuda.Stream().cuda_stream
        g = make_slab(n, tile, r, nranks, faces, 0.0, comm).mg_setup(levels, 1, 0.5, 16)
        g.set_vector(B.B, local_part(g, b), stream=s)
        it, rel, ok = g.pcg_solve(B.PC_MG, 1.0, B.PAIR_SYMMETRIC, 1e-8, 2000, stream=s)
        return it, ok, g.get_vector(B.X, stream=s)
    res = run_threads(nranks, rank_fn)
    its = {r[0] for r in res}
    assert ok1 and len(its) == 1 and all(r[1] for r in res)
    assert abs(its.pop() - it1) <= 1
    assert O.relres(pb, np.concatenate([r[2] for r in res], axis=0), b) < 2e-8


def test_multirank_validation():
    n, tile = (128, 128), (64, 64)
    g = make_slab(n, tile, 0, 2)                       # no communicator: staged use only
    with pytest.raises(B.SweepError):
        g.sor_sweep([1.5], 2, 0)
    with pytest.raises(B.SweepError):
        g.pcg_solve(B.PC_ILU0)
    with pytest.raises(B.SweepError):
        g.residual_norm()
    hub = parallel.ThreadHub(2)
    comm = parallel.host_comm(1, 2, hub.endpoint(1))
    with pytest.raises(B.SweepError):                  # communicator rank differs from the slab's
        make_slab(n, tile, 0, 2, comm=comm)
