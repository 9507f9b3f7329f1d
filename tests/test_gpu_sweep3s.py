"""GPU parity of the streaming 3D engine (k_sweep3s, csrc/sweep3s.cuh) against the oracle.

The library dispatches it for boxes at least 64 long in x (k_sweep3 cannot stage them); the
subprocess test forces it (SW_SWEEP3=new) on the shapes k_sweep3 handles by default, so both
engines stay bitwise equal to the oracle on every shape they may run."""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle as O
from paper_1008_3699_b200 import gen
from tests.gpu_helpers import make_grid, rand_faces, rel_maxdiff

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (n, tile, variable coefficients?, beta, omega): boxes long in x, every start-face coupling
# pattern (interior, boundary and one-box-thick directions), per-direction omega
LONG = [
    ((128, 16, 8), (64, 8, 4), True, 0.0, [1.0]),
    ((128, 16, 8), (64, 8, 4), True, 0.1, list(0.6 + 0.15 * np.arange(8))),
    ((256, 8, 8), (128, 4, 4), False, 0.1, list(1.9 - 0.1 * np.arange(8))),
    ((64, 24, 12), (64, 6, 3), True, 0.0, [1.2]),          # one box along x, ragged y/z counts
    ((192, 8, 4), (64, 8, 4), True, 0.0, [1.3]),           # one box in y and z
]


@pytest.mark.parametrize("n,tile,var,beta,omega", LONG)
def test_long_box_sweep_matches_oracle(gpu_lib, n, tile, var, beta, omega):
    faces = rand_faces(n, 7) if var else None
    pb = O.tiled(n, tile, faces=faces, beta=beta)
    g = make_grid(gpu_lib, n, tile, faces, beta)
    x = gen.uniform_field(1, gen.STREAM_X0, pb.shape)
    b = gen.uniform_field(1, gen.STREAM_RHS, pb.shape)
    g.set_vector(gpu_lib.X, x)
    g.set_vector(gpu_lib.B, b)
    phase = 0
    for k in range(2 ** len(n) + 2):                         # every direction of the cycle, twice for two
        x = O.sweep(pb, omega, x, b, phase=k)
        phase = g.sor_sweep(omega, 1, phase)
        got = g.get_vector(gpu_lib.X)
        assert np.array_equal(got, x), (k, rel_maxdiff(got, x))
    g.check()


@pytest.mark.parametrize("n,tile,var,beta", [((128, 16, 8), (64, 8, 4), True, 0.0),
                                             ((256, 8, 8), (128, 4, 4), False, 0.2)])
def test_long_box_ilu_and_ssor_apply_match_oracle(gpu_lib, n, tile, var, beta):
    faces = rand_faces(n, 17) if var else None
    pb = O.tiled(n, tile, faces=faces, beta=beta)
    g = make_grid(gpu_lib, n, tile, faces, beta)
    r = gen.uniform_field(5, gen.STREAM_TEST, pb.shape)
    g.ilu0_factor(0)
    inv = O.ilu0_factor(pb, phase=0)
    g.set_vector(gpu_lib.R, r)
    for pairing in (0, 1):
        g.ilu_apply(g.ptr(gpu_lib.R), g.ptr(gpu_lib.Z), pairing)
        assert np.array_equal(g.get_vector(gpu_lib.Z), O.ilu_apply(pb, inv, r, pairing))
        g.ssor_apply(1.3, g.ptr(gpu_lib.R), g.ptr(gpu_lib.Z), pairing)
        assert np.array_equal(g.get_vector(gpu_lib.Z), O.ssor_apply(pb, 1.3, r, pairing))
    g.check()


def test_long_box_pcg_iterations_match_oracle(gpu_lib):
    n, tile = (128, 16, 12), (64, 8, 4)
    ring = tuple(v + 2 for v in reversed(n))
    faces = O.faces_from_k(n, gen.lognormal_k(0, ring, 0.5), (1.0, 0.1, 0.01))
    pb = O.tiled(n, tile, faces=faces)
    g = make_grid(gpu_lib, n, tile, faces)
    b = gen.uniform_field(0, gen.STREAM_RHS, pb.shape) / float((n[0] + 1) ** 2)
    g.set_vector(gpu_lib.B, b)
    it, rel, ok = g.pcg_solve(2, 1.0, 0, 1e-8, 5000)
    _, ito, _, oko = O.pcg(pb, b, precond=2, omega=1.0, pairing=0, rtol=1e-8, maxit=5000)
    assert ok and oko and abs(it - ito) <= 1, (it, ito)
    assert O.relres(pb, g.get_vector(gpu_lib.X), b) < 2e-8


def test_streaming_engine_forced_on_short_boxes():
    """The 3D parity cases of test_gpu_parity.py (32 x 8 x 4, 16 x 8 x 4 and 4 x 6 x 3 boxes; sweeps,
    ILU / SSOR applications, PCG) with the streaming engine forced in place of k_sweep3."""
    env = dict(os.environ, SW_SWEEP3="new")
    sel = "n13 or n14 or n15 or n16 or n11-tile11 or n12-tile12 or n8-tile8 or n9-tile9 or n10-tile10"
    res = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider",
                          os.path.join(ROOT, "tests", "test_gpu_parity.py"), "-k", sel],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-2000:]
    assert " passed" in res.stdout and "failed" not in res.stdout, res.stdout[-2000:]
