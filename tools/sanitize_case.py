"""One small invocation of every hot-path kernel, for compute-sanitizer (racecheck / synccheck /
memcheck; SURVEY.md §5 race detection).  Run as ``python tools/sanitize_case.py [group]`` under
``compute-sanitizer --tool <tool>``; tests/test_gpu_sanitizer.py does that and fails on any report.

Groups keep each sanitizer run short: ``2d`` (k_sweep2p, k_sweep2v SOR and TRI, k_tri2t),
``3d`` (k_sweep3 SOR and TRI, k_tri3t, k_pspmv3_zm), ``generic`` (k_generic: 1D, odd boxes, the ILU
factor), ``blas`` (the PCG vector kernels and k_finish_sum through a short PCG), ``mg`` (one V-cycle).
No oracle: the parity tests check the values; this only drives the kernels."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_1008_3699_b200 import binding as B, gen  # noqa: E402


def faces_for(n, seed):
    out = []
    for a in range(len(n)):
        m = list(n)
        m[a] += 1
        shape = tuple(reversed(m))
        out.append(0.5 + 1.5 * gen.unit(seed, gen.STREAM_TEST + a, int(np.prod(shape))).reshape(shape))
    return out


def grid(n, tile, var, beta=0.0):
    g = B.Grid(len(n), n, B.COEF_FACES if var else B.COEF_POISSON, beta).decompose(tile)
    if var:
        g.set_faces_global(faces_for(n, 3))
    shape = tuple(reversed(n))
    g.set_vector(B.X, gen.uniform_field(1, gen.STREAM_X0, shape))
    g.set_vector(B.B, gen.uniform_field(1, gen.STREAM_RHS, shape) / float((n[0] + 1) ** 2))
    g.set_vector(B.R, gen.uniform_field(2, gen.STREAM_TEST, shape))
    return g


def precond_all(g):
    for pairing in (B.PAIR_SYMMETRIC, B.PAIR_PAPER):
        g.ssor_apply(1.2, g.ptr(B.R), g.ptr(B.Z), pairing)
    g.ilu0_factor(0)
    for pairing in (B.PAIR_SYMMETRIC, B.PAIR_PAPER):
        g.ilu_apply(g.ptr(B.R), g.ptr(B.Z), pairing)


def run(group):
    if group == "2d":
        for var in (False, True):
            g = grid((192, 128), (64, 64), var)
            g.sor_sweep([1.3], 4, 0)
            precond_all(g)
            g.check()
    elif group == "3d":
        for var in (False, True):
            g = grid((64, 16, 8), (32, 8, 4), var)
            g.sor_sweep([1.1], 8, 0)
            precond_all(g)
            g.pcg_solve(B.PC_ILU0, 1.0, B.PAIR_SYMMETRIC, 1e-6, 3)
            g.check()
    elif group == "generic":
        g = grid((100,), (10,), True)
        g.sor_sweep([1.5], 2, 0)
        precond_all(g)
        g = grid((30, 24), (10, 8), True, 0.1)
        g.sor_sweep([1.2], 4, 0)
        precond_all(g)
        g = grid((15, 12, 12), (5, 4, 6), True)
        g.sor_sweep([1.0], 2, 0)
        precond_all(g)
        g.check()
    elif group == "blas":
        g = grid((128, 128), (64, 64), True)
        g.pcg_solve(B.PC_SSOR, 1.0, B.PAIR_PAPER, 1e-6, 4)
        g.residual_norm()
        g.check()
    elif group == "mg":
        g = grid((128, 128), (32, 32), True).mg_setup(3, 1, 0.5, 2)
        g.mg_apply(g.ptr(B.R), g.ptr(B.Z))
        g.check()
    else:
        raise SystemExit(f"unknown group {group}")
    import torch
    torch.cuda.synchronize()
    print(f"sanitize case {group} done")


if __name__ == "__main__":
    run(sys.argv[1] if len(sys.argv) > 1 else "2d")
