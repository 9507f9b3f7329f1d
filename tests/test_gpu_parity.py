"""GPU parity: the CUDA path (through the C ABI) against the oracle on the same seeded
inputs.  Bar (north_star): 1e-12 relative max-norm per sweep; the sweep kernels mirror
the oracle's operation order, so we assert exact equality (==, i.e. up to the sign of
zero) and report the max-norm too."""
import numpy as np
import pytest

import oracle as O
from paper_1008_3699_b200 import gen
from tests.gpu_helpers import make_grid, rand_faces, rel_maxdiff

pytestmark = pytest.mark.gpu


def _inputs(pb, seed):
    x0 = gen.uniform_field(seed, gen.STREAM_X0, pb.shape)
    b = gen.uniform_field(seed, gen.STREAM_RHS, pb.shape)
    return x0, b


CASES = [
    # (n, tile, variable coefficients?, beta, omega)
    ((256, 256), (64, 64), False, 0.0, [1.975848]),                  # config 2 shape
    ((256, 256), (64, 64), True, 0.0, [1.0]),                       # config 3 law, small
    ((320, 192), (64, 64), False, 0.1, [0.7, 1.3, 1.1, 1.6]),       # Poisson kernel, per-direction omega, beta
    ((64, 64), (64, 64), False, 0.0, [1.9]),                        # Poisson kernel, one box
    ((128, 64), (64, 64), False, 0.0, [1.99]),                      # Poisson kernel, one tile row
    ((64, 192), (64, 64), False, 0.3, [0.5]),                       # Poisson kernel, one tile column
    ((192, 320), (64, 64), True, 0.1, [0.7, 1.3, 1.1, 1.6]),        # odd tile counts, per-direction omega
    ((130, 66), (26, 22), False, 0.0, [1.5]),                       # ragged tiles, 5x3 boxes
    ((64, 64), (64, 64), True, 0.0, [1.2]),                         # one box
    ((1024,), (256,), False, 0.0, [2 / (1 + np.sin(np.pi / 1025))]),  # config 1
    ((100,), (10,), True, 0.05, [0.9, 1.4]),                         # 1D faces, per-direction omega
    ((32, 32, 32), (16, 8, 8), True, 0.0, [1.0]),                   # 3D, boxes long in x
    ((24, 16, 16), (8, 8, 8), False, 0.0, [1.3]),
    ((12, 12, 12), (4, 6, 3), True, 0.2, list(0.6 + 0.15 * np.arange(8))),
    ((64, 32, 16), (32, 8, 4), True, 0.0, [1.0]),                   # 3D kernel, C5-shaped boxes
    ((64, 16, 16), (32, 8, 4), False, 0.1, list(1.9 - 0.1 * np.arange(8))),   # Poisson, per-direction omega
    ((32, 8, 4), (32, 8, 4), True, 0.0, [1.3]),                     # one box
    ((15, 12, 12), (5, 4, 6), True, 0.0, [1.1]),                    # odd box edge: generic kernel
]


@pytest.mark.parametrize("n,tile,var,beta,omega", CASES)
def test_sor_sweep_matches_oracle(gpu_lib, n, tile, var, beta, omega):
    faces = rand_faces(n, 7) if var else None
    pb = O.tiled(n, tile, faces=faces, beta=beta)
    g = make_grid(gpu_lib, n, tile, faces, beta)
    x0, b = _inputs(pb, 1)
    g.set_vector(gpu_lib.X, x0)
    g.set_vector(gpu_lib.B, b)
    x = x0
    phase = 0
    for k in range(2 ** len(n) + 2):
        x = O.sweep(pb, omega, x, b, phase=k)
        phase = g.sor_sweep(omega, 1, phase)
        got = g.get_vector(gpu_lib.X)
        err = rel_maxdiff(got, x)
        assert err <= 1e-12, (k, err)
        assert np.array_equal(got, x), (k, err)
    g.check()


def test_multi_sweep_call_and_phase(gpu_lib):
    n, tile = (128, 192), (64, 64)
    pb = O.tiled(n, tile)
    g = make_grid(gpu_lib, n, tile)
    x0, b = _inputs(pb, 2)
    g.set_vector(gpu_lib.X, x0)
    g.set_vector(gpu_lib.B, b)
    ph = g.sor_sweep([1.8], 9, 5)
    assert ph == 14
    x = x0
    for k in range(5, 14):
        x = O.sweep(pb, [1.8], x, b, phase=k)
    assert np.array_equal(g.get_vector(gpu_lib.X), x)


def test_faces_from_k_matches_oracle(gpu_lib):
    for n in [(40, 24), (12, 10, 8), (30,)]:
        ring = tuple(v + 2 for v in reversed(n))
        kr = gen.lognormal_k(3, ring, 1.0)
        scale = (1.0, 0.1, 0.01)[: len(n)]
        F = O.faces_from_k(n, kr, scale)
        # k layout for the slab: slab axis (numpy axis 0) gets one more dummy layer per side
        pad = [(0, 0)] * len(n)
        pad[0] = (1, 1)
        k_ext = np.pad(kr, pad, constant_values=1.0)
        tile = tuple(v // 2 if v % 2 == 0 else v for v in n)
        pb = O.tiled(n, tile, faces=F)
        g = gpu_lib.Grid(len(n), n, gpu_lib.COEF_FACES).decompose(tile)
        g.set_coefficients_k(k_ext, scale)
        x0, b = _inputs(pb, 4)
        g.set_vector(gpu_lib.X, x0)
        g.set_vector(gpu_lib.B, b)
        g.sor_sweep([1.1], 1, 0)
        assert np.array_equal(g.get_vector(gpu_lib.X), O.sweep(pb, [1.1], x0, b, phase=0))


TRI_CASES = [((64, 64), (16, 16), True, 0.0), ((96, 64), (32, 16), True, 0.0), ((256, 256), (64, 64), True, 0.0),
             ((16, 16, 16), (8, 8, 8), True, 0.0), ((20, 12, 8), (10, 4, 4), True, 0.0), ((200,), (40,), True, 0.0),
             # 64 x 64 boxes: the fast 2D engine (unit and variable coefficients, beta, one box, strips)
             ((192, 128), (64, 64), False, 0.0), ((128, 320), (64, 64), True, 0.3), ((64, 64), (64, 64), True, 0.0),
             ((320, 64), (64, 64), False, 0.1), ((64, 256), (64, 64), True, 0.0),
             # 3D kernel (forward solves; coupled-set phase of the transposed solve on the generic kernel)
             ((64, 32, 16), (32, 8, 4), True, 0.0), ((32, 16, 8), (16, 8, 4), False, 0.2)]


@pytest.mark.parametrize("n,tile,var,beta", TRI_CASES)
def test_ilu_and_ssor_apply_match_oracle(gpu_lib, n, tile, var, beta):
    faces = rand_faces(n, 17) if var else None
    pb = O.tiled(n, tile, faces=faces, beta=beta)
    g = make_grid(gpu_lib, n, tile, faces, beta)
    r = gen.uniform_field(5, gen.STREAM_TEST, pb.shape)
    g.ilu0_factor(0)
    inv = O.ilu0_factor(pb, phase=0)
    got_inv = g.get_vector(gpu_lib.INVD)
    assert np.array_equal(got_inv, inv)
    g.set_vector(gpu_lib.R, r)
    for pairing in (0, 1):
        g.ilu_apply(g.ptr(gpu_lib.R), g.ptr(gpu_lib.Z), pairing)
        z = g.get_vector(gpu_lib.Z)
        zo = O.ilu_apply(pb, inv, r, pairing)
        assert rel_maxdiff(z, zo) <= 1e-12
        assert np.array_equal(z, zo)
        for w in (1.0, 1.4):
            g.ssor_apply(w, g.ptr(gpu_lib.R), g.ptr(gpu_lib.Z), pairing)
            z = g.get_vector(gpu_lib.Z)
            zo = O.ssor_apply(pb, w, r, pairing)
            assert np.array_equal(z, zo)
    g.check()


@pytest.mark.parametrize("n,tile,var,pc", [((64, 64), (16, 16), False, 2), ((256, 256), (64, 64), False, 2),
                                           ((256, 256), (64, 64), True, 2), ((128, 128), (32, 32), True, 1),
                                           ((16, 16, 16), (8, 8, 8), True, 2), ((128, 64), (32, 32), False, 0),
                                           ((192, 256), (64, 64), True, 1), ((256, 128), (64, 64), False, 1),
                                           # 3D ragged for the z-marching fused update + SpMV (k_pspmv3_zm): n1 not
                                           # a multiple of its 8-row tile, n2 not a multiple of its 8-plane chunk
                                           ((24, 12, 10), (8, 6, 5), False, 2), ((24, 12, 10), (8, 6, 5), True, 2),
                                           ((40, 20, 18), (8, 4, 6), True, 1), ((24, 13, 11), (24, 13, 11), True, 0)])
def test_pcg_iterations_match_oracle(gpu_lib, n, tile, var, pc):
    faces = None
    if var:
        ring = tuple(v + 2 for v in reversed(n))
        faces = O.faces_from_k(n, gen.lognormal_k(0, ring, 1.0))
    pb = O.tiled(n, tile, faces=faces)
    g = make_grid(gpu_lib, n, tile, faces)
    b = gen.uniform_field(0, gen.STREAM_RHS, pb.shape) / float((n[0] + 1) ** 2)
    g.set_vector(gpu_lib.B, b)
    it, rel, ok = g.pcg_solve(pc, 1.0, 0, 1e-8, 5000)
    xo, ito, relo, oko = O.pcg(pb, b, precond=pc, omega=1.0, pairing=0, rtol=1e-8, maxit=5000)
    assert ok and oko
    assert abs(it - ito) <= 1, (it, ito)
    x = g.get_vector(gpu_lib.X)
    assert O.relres(pb, x, b) < 2e-8


@pytest.mark.parametrize("n,tile,var,pc,pairing,mode", [
    ((64, 64), (16, 16), False, 2, 1, -1),          # PAPER pairing: flexible beta chosen automatically
    ((64, 64), (16, 16), True, 1, 1, -1),
    ((16, 16, 16), (8, 8, 8), True, 2, 1, -1),
    ((32, 16, 8), (16, 8, 4), True, 2, 1, -1),
    ((64, 64), (16, 16), True, 2, 0, 1),            # flexible beta forced with the SYMMETRIC pairing
])
def test_flexible_pcg_matches_oracle(gpu_lib, n, tile, var, pc, pairing, mode):
    """Flexible (Polak-Ribiere) PCG, which the nonsymmetric PAPER pairing needs (SURVEY §8(c)
    C-PCG): iteration count within 1 of the oracle's or_pcg(flexible=1), solution to 2e-8."""
    faces = None
    if var:
        ring = tuple(v + 2 for v in reversed(n))
        faces = O.faces_from_k(n, gen.lognormal_k(0, ring, 1.0))
    pb = O.tiled(n, tile, faces=faces)
    g = make_grid(gpu_lib, n, tile, faces).set_pcg_flexible(mode)
    b = gen.uniform_field(0, gen.STREAM_RHS, pb.shape) / float((n[0] + 1) ** 2)
    g.set_vector(gpu_lib.B, b)
    it, rel, ok = g.pcg_solve(pc, 1.0, pairing, 1e-8, 5000)
    xo, ito, relo, oko = O.pcg(pb, b, precond=pc, omega=1.0, pairing=pairing, flexible=True, rtol=1e-8, maxit=5000)
    assert ok and oko
    assert abs(it - ito) <= 1, (it, ito)
    assert O.relres(pb, g.get_vector(gpu_lib.X), b) < 2e-8


def test_pcg_flexible_mode_validation(gpu_lib):
    g = make_grid(gpu_lib, (64, 64), (16, 16))
    with pytest.raises(gpu_lib.SweepError):
        g.set_pcg_flexible(2)
