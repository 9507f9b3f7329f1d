"""Model problem of the paper's experiments (TEST INFRASTRUCTURE ONLY).

PAPER:1906-1934: Laplace's equation on [0,1]^d with u = prod_i x_i on the boundary,
u^0 = 0, stop when the L1 error against the exact solution prod_i x_i is below
1e-3 (3D: 1e-2).  Readings: resolution R counts nodes including the
boundary (n = R - 2, R-1), the L1 normaliser is R^d in 1D/3D and 3 R^2 in 2D (R-2),
every directional pass counts as one iteration (R-3).

The h^2-scaled 2d+1 point Laplacian has unit face coefficients, so the boundary
fold of PAPER:215 (f_1 = c_1 u_0 + f_1 ...) adds the boundary value of every
boundary neighbour to b.
"""
from __future__ import annotations

import numpy as np

from . import Problem, balanced_bounds, sor_lex, sweep


def model_problem(dim: int, R: int, parts=None):
    n = R - 2
    h = 1.0 / (R - 1)
    coords = np.arange(1, n + 1) * h
    parts = parts or [1] * dim
    pb = Problem(tuple([n] * dim), tuple(balanced_bounds(n, p) for p in parts))
    # exact solution at interior nodes, numpy order (z, y, x)
    grids = np.meshgrid(*([coords] * dim), indexing="ij")   # grids[a] varies along numpy axis a
    exact = np.ones([n] * dim)
    for gr in grids:
        exact = exact * gr
    # boundary fold: b = sum over boundary neighbours of u_boundary (face coefficient 1)
    b = np.zeros([n] * dim)
    full = np.arange(0, n + 2) * h                            # all node coordinates incl. boundary
    for ax in range(dim):
        for side, idx_b in ((0, 0), (-1, n + 1)):
            # neighbour in the boundary layer along numpy axis ax
            sl = [slice(None)] * dim
            sl[ax] = side
            bcoord = full[idx_b]
            val = np.ones([n] * dim)
            for a2, gr in enumerate(grids):
                val = val * (bcoord if a2 == ax else gr)
            b[tuple(sl)] += val[tuple(sl)]
    return pb, b, exact


def l1_error(u, exact, R: int, dim: int) -> float:
    s = float(np.abs(u - exact).sum())
    return s / (3.0 * R * R) if dim == 2 else s / float(R ** dim)


def run_until(dim, R, step, tol, maxit=100000):
    """Iterate `step(k, u) -> u` from u=0 until the L1 error < tol; returns (iterations, L1)."""
    pb, b, exact = model_problem(dim, R)
    u = np.zeros(pb.shape)
    for k in range(maxit):
        u = step(k, u, pb, b)
        e = l1_error(u, exact, R, dim)
        if e < tol:
            return k + 1, e
    return None, e


def run_decomposed(dim, R, parts, omega, tol, override_seq=None, maxit=100000):
    pb, b, exact = model_problem(dim, R, parts)
    u = np.zeros(pb.shape)
    for k in range(maxit):
        ov = -1 if override_seq is None else override_seq[k % len(override_seq)]
        u = sweep(pb, omega, u, b, phase=k, override=ov)
        e = l1_error(u, exact, R, dim)
        if e < tol:
            return k + 1, e
    return None, e


def run_lex(dim, R, omegas, corners, tol, maxit=100000):
    """Classical sweeps: iteration k uses corner corners[k % len] and omega omegas[k % len]."""
    pb, b, exact = model_problem(dim, R)
    u = np.zeros(pb.shape)
    for k in range(maxit):
        u = sor_lex(pb, omegas[k % len(omegas)], u, b, corners[k % len(corners)])
        e = l1_error(u, exact, R, dim)
        if e < tol:
            return k + 1, e
    return None, e
