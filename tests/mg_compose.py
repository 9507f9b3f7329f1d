"""The oracle-side composition of the multigrid preconditioner (DESIGN R-17/R-19):
piecewise-constant aggregation, Galerkin face sums, m-step SGS smoothing and the V/W-cycle, built
from oracle calls and numpy.  TEST INFRASTRUCTURE: used by tests/test_gpu_mg.py as the expected
value and pinned against dense linear algebra (P^T A P, a dense-matrix V-cycle) in
tests/test_oracle_pins.py."""
import numpy as np

import oracle as O


# ---- the oracle-side V-cycle (numpy + oracle calls; sums in the order DESIGN R-19 fixes: pairwise
# along the coarsened axes, ascending)
def _pairs(v, ax):
    return np.take(v, np.arange(0, v.shape[ax], 2), axis=ax) + np.take(v, np.arange(1, v.shape[ax], 2), axis=ax)


def coarsen_faces(faces, n, mask):
    dim = len(n)
    out = []
    for a in range(dim):
        f = np.ones(O.face_shape(n, a)) if faces is None else np.asarray(faces[a])
        ax = dim - 1 - a                                   # numpy axis of grid axis a
        g = np.take(f, np.arange(0, f.shape[ax], 2), axis=ax) if (mask >> a) & 1 else f
        for b in range(dim):                               # the other coarsened axes, ascending
            if b != a and (mask >> b) & 1:
                g = _pairs(g, dim - 1 - b)
        out.append(g)
    return tuple(out)


def restrict(r, mask):
    dim = r.ndim
    for a in range(dim):
        if (mask >> a) & 1:
            r = _pairs(r, dim - 1 - a)
    return r


def prolong(xc, mask):
    dim = xc.ndim
    for a in range(dim):
        if (mask >> a) & 1:
            xc = np.repeat(xc, 2, axis=dim - 1 - a)
    return xc


def coarse_tile(t, nc):
    t = min(t, nc)
    while nc % t:
        t -= 1
    return t


def build_levels(n, tile, faces, beta, levels, mask):
    lv = [(tuple(n), tuple(tile), faces, beta)]
    k = bin(mask).count("1")
    for _ in range(levels - 1):
        n0, t0, f0, b0 = lv[-1]
        nc = tuple(v // 2 if (mask >> a) & 1 else v for a, v in enumerate(n0))
        tc = tuple(coarse_tile(t, v) for t, v in zip(t0, nc))
        lv.append((nc, tc, coarsen_faces(f0, n0, mask), b0 * 2 ** k))
    return [O.tiled(nn, tt, faces=ff, beta=bb) for nn, tt, ff, bb in lv]


def smooth(pb, r, m, theta):
    z = O.ssor_apply(pb, 1.0, r, 0)
    for _ in range(m - 1):
        z = z + O.ssor_apply(pb, 1.0, r - theta * O.apply_A(pb, z), 0)
    return theta * z


def vcycle(pbs, lev, r, nu, theta, nu_c, sc=1.0, mask=7, gamma=1):
    pb = pbs[lev]
    if lev == len(pbs) - 1:
        return smooth(pb, r, nu_c, theta)
    x = smooth(pb, r, nu, theta)
    rc = restrict(r - O.apply_A(pb, x), mask)
    xc = vcycle(pbs, lev + 1, rc, nu, theta, nu_c, sc, mask, gamma)
    if gamma == 2 and lev + 1 < len(pbs) - 1:         # W-cycle: second coarse cycle on the coarse residual
        xc = xc + vcycle(pbs, lev + 1, rc - O.apply_A(pbs[lev + 1], xc), nu, theta, nu_c, sc, mask, gamma)
    x = x + sc * prolong(xc, mask)
    return x + smooth(pb, r - O.apply_A(pb, x), nu, theta)
