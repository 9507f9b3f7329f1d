"""The omega search on the GPU: the library counter `omega.sweeps_to_tol`
(decomposed SOR sweeps through the C ABI, relative residual checked every 10 sweeps) gives the
same sweep counts as the same loop over the oracle, for one omega and for per-direction
omegas, so a search over the library finds the oracle's optimum."""
import numpy as np
import pytest

import oracle as O
from paper_1008_3699_b200 import binding as B, gen, omega as OM
from tests.gpu_helpers import make_grid

pytestmark = pytest.mark.gpu

N, TILE = (128, 128), (64, 64)


def oracle_count(pb, b, omega, tol=1e-8, maxit=4000, every=10):
    x = np.zeros(pb.shape)
    ph, n = 0, 0
    while n < maxit:
        for _ in range(every):
            x = O.sweep(pb, omega, x, b, ph)
            ph += 1
        n += every
        r = O.relres(pb, x, b)
        if not np.isfinite(r):
            return None
        if r < tol:
            return n
    return None


@pytest.mark.parametrize("omega", [[1.9], [1.95], [1.93, 1.9, 1.92, 1.95]])
def test_library_counts_equal_oracle_counts(omega):
    pb = O.tiled(N, TILE)
    b = gen.uniform_field(1, gen.STREAM_RHS, pb.shape) / float((N[0] + 1) ** 2)
    g = make_grid(B, N, TILE)
    g.set_vector(B.B, b)
    got = OM.sweeps_to_tol(g, omega, 1e-8, 4000, 10)
    want = oracle_count(pb, b, omega)
    assert got == want and got is not None


def test_search_on_the_library_finds_the_oracle_optimum():
    pb = O.tiled(N, TILE)
    b = gen.uniform_field(2, gen.STREAM_RHS, pb.shape) / float((N[0] + 1) ** 2)
    g = make_grid(B, N, TILE)
    g.set_vector(B.B, b)
    w_lib, c_lib, t_lib = OM.grid_search(lambda v: OM.sweeps_to_tol(g, v, 1e-8, 4000, 10), 1.90, 1.98, 0.02)
    w_or, c_or, t_or = OM.grid_search(lambda v: oracle_count(pb, b, v), 1.90, 1.98, 0.02)
    assert t_lib == t_or
    assert (w_lib, c_lib) == (w_or, c_or)


def test_config1_sweep_count_equals_oracle():
    """Config 1 (1D Poisson, n = 1024, 4 boxes of 256, omega_opt): the number of decomposed SOR
    sweeps to a relative residual of 1e-8 (checked after every sweep) equals the oracle's."""
    n, tile = (1024,), (256,)
    w = [OM.omega_opt_poisson(n[0])]
    pb = O.tiled(n, tile)
    b = gen.uniform_field(0, gen.STREAM_RHS, pb.shape) / float((n[0] + 1) ** 2)
    g = make_grid(B, n, tile)
    g.set_vector(B.B, b)
    got = OM.sweeps_to_tol(g, w, 1e-8, 100000, 1)
    want = oracle_count(pb, b, w, 1e-8, 100000, 1)
    assert got == want and got is not None
