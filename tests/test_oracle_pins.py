"""Pins for the oracle pieces that had none, each against an
independent definition (-m "not gpu"):

* ``or_relres`` / ``or_apply_A``: ||b - A x||_2 / ||b||_2 with A assembled here in numpy straight
  from the stencil definition (a_P = sum of faces + beta, off-diagonal
  -c on each face between two interior nodes), not through the oracle.
* ``or_pcg``: iterate for iterate against textbook PCG written in numpy on that dense A with the
  dense preconditioner matrix -- the Polak-Ribiere beta = z+.(r+ - r)/(r.z) for ``flexible`` and
  beta = (r+.z+)/(r.z) otherwise (SURVEY §8(c) C-PCG).
* the test-side multigrid composition (``tests/mg_compose.py``, DESIGN R-19): coarse faces
  against the dense Galerkin product P^T A P with piecewise-constant P built from the aggregation
  definition; restriction / prolongation against P^T and P; one V- and W-cycle against the same
  cycle written with dense matrices.
Each test states which plausible mistake it catches."""
import numpy as np
import pytest

import oracle as O
from paper_1008_3699_b200 import gen
from tests.mg_compose import build_levels, coarsen_faces, prolong, restrict, vcycle


def rand_faces(n, seed, lo=0.5, hi=2.0):
    return tuple(lo + (hi - lo) * gen.unit(seed, gen.STREAM_TEST + a, int(np.prod(O.face_shape(n, a)))).reshape(
        O.face_shape(n, a)) for a in range(len(n)))


def assemble_A(n, faces, beta):
    """Dense A of the 2d+1-point operator from its definition (x fastest numbering):
    A_pp = sum of the 2d faces of p + beta, A_pq = -c_pq for interior neighbours."""
    dim = len(n)
    shape = tuple(reversed(n))
    N = int(np.prod(n))
    idx = np.arange(N).reshape(shape)
    diag = np.full(shape, float(beta))
    A = np.zeros((N, N))
    for a in range(dim):
        ax = dim - 1 - a
        F = np.ones(O.face_shape(n, a)) if faces is None else np.asarray(faces[a], dtype=np.float64)
        lower = np.take(F, np.arange(0, n[a]), axis=ax)        # face between p - e_a and p
        upper = np.take(F, np.arange(1, n[a] + 1), axis=ax)    # face between p and p + e_a
        diag = diag + lower + upper
        inner = np.take(F, np.arange(1, n[a]), axis=ax).ravel()
        i0 = np.take(idx, np.arange(0, n[a] - 1), axis=ax).ravel()
        i1 = np.take(idx, np.arange(1, n[a]), axis=ax).ravel()
        A[i0, i1] = -inner
        A[i1, i0] = -inner
    A[np.arange(N), np.arange(N)] = diag.ravel()
    return A


def precond_inverse(apply, N, shape):
    """Dense P^-1 (columns = images of unit vectors)."""
    M = np.empty((N, N))
    for j in range(N):
        e = np.zeros(N)
        e[j] = 1.0
        M[:, j] = apply(e.reshape(shape)).ravel()
    return M


# ------------------------------------------------------------------------------- or_relres
@pytest.mark.parametrize("n,beta", [((37,), 0.0), ((9, 7), 0.0), ((6, 5, 4), 0.3)])
def test_relres_and_apply_A_match_dense_definition(n, beta):
    """Catches: a dropped sqrt (relres^2), a missing / wrong ||b|| normaliser, a wrong sign of the
    residual, a missing face in a_P or a transposed face index in A x."""
    F = rand_faces(n, 91)
    pb = O.tiled(n, n, faces=F, beta=beta)
    A = assemble_A(n, F, beta)
    N = pb.size
    x = gen.uniform(4, gen.STREAM_TEST, N)
    b = gen.uniform(5, gen.STREAM_RHS, N) * 3.0
    Ax = A @ x
    assert np.max(np.abs(O.apply_A(pb, x.reshape(pb.shape)).ravel() - Ax)) <= 1e-13 * np.max(np.abs(Ax))
    for xx in (x, 0.5 * np.linalg.solve(A, b) + 0.01 * x):          # relres ~ O(1) and ~ 0.5
        want = np.linalg.norm(b - A @ xx) / np.linalg.norm(b)
        got = O.relres(pb, xx.reshape(pb.shape), b.reshape(pb.shape))
        assert abs(got - want) <= 1e-12 * want, (got, want)
        assert abs(want ** 2 - want) > 1e-3 and abs(np.linalg.norm(b) - 1.0) > 1e-3   # the test can tell
    # exact solution -> ~0; b = 0 -> the unnormalised norm (documented behaviour)
    xs = np.linalg.solve(A, b)
    assert O.relres(pb, xs.reshape(pb.shape), b.reshape(pb.shape)) < 1e-13
    got0 = O.relres(pb, x.reshape(pb.shape), np.zeros(pb.shape))
    assert abs(got0 - np.linalg.norm(Ax)) <= 1e-12 * np.linalg.norm(Ax)


# ------------------------------------------------------------------------------- or_pcg
def textbook_pcg(A, Minv, b, iters, flexible):
    """Textbook PCG from x0 = 0; flexible = Polak-Ribiere beta = z+.(r+ - r)/(r.z)."""
    x = np.zeros_like(b)
    r = b.copy()
    z = Minv @ r
    p = z.copy()
    rz = r @ z
    xs = []
    for _ in range(iters):
        q = A @ p
        al = rz / (p @ q)
        rold = r.copy()
        x = x + al * p
        r = r - al * q
        xs.append(x.copy())
        z = Minv @ r
        rzn = r @ z
        be = (z @ (r - rold)) / rz if flexible else rzn / rz
        rz = rzn
        p = z + be * p
    return xs


@pytest.mark.parametrize("precond,pairing,flexible", [(2, 1, True), (1, 1, True), (2, 0, False), (1, 0, False),
                                                      (2, 0, True)])
def test_pcg_iterates_match_textbook_pcg(precond, pairing, flexible):
    """or_pcg after k = 1..6 iterations equals textbook PCG's x_k (1e-11).  With the nonsymmetric
    PAPER pairing the flexible and the standard beta give iterates that differ by >> 1e-11 from
    the third iteration on, so a standard beta in the flexible branch (or a wrong Polak-Ribiere
    formula: z+.r+ / r.z, or r+ - r with the sign flipped) fails."""
    n, tile = (12, 10), (4, 5)
    F = rand_faces(n, 83)
    pb = O.tiled(n, tile, faces=F)
    A = assemble_A(n, F, 0.0)
    N = pb.size
    b = gen.uniform(1, gen.STREAM_RHS, N)
    if precond == 2:
        inv = O.ilu0_factor(pb, phase=0)
        Minv = precond_inverse(lambda r: O.ilu_apply(pb, inv, r, pairing), N, pb.shape)
    else:
        Minv = precond_inverse(lambda r: O.ssor_apply(pb, 1.3, r, pairing), N, pb.shape)
    ref = textbook_pcg(A, Minv, b, 6, flexible)
    other = textbook_pcg(A, Minv, b, 6, not flexible)
    for k in range(1, 7):
        x, it, rel, ok = O.pcg(pb, b.reshape(pb.shape), precond=precond, omega=1.3, pairing=pairing,
                               flexible=flexible, rtol=1e-300, maxit=k)
        assert it == k and not ok
        scale = np.max(np.abs(ref[k - 1]))
        assert np.max(np.abs(x.ravel() - ref[k - 1])) <= 1e-11 * scale, k
        want_rel = np.linalg.norm(b - A @ ref[k - 1]) / np.linalg.norm(b)
        assert abs(rel - want_rel) <= 1e-8 * want_rel + 1e-14      # recursive vs true residual
    if pairing == 1:
        assert np.max(np.abs(other[3] - ref[3])) > 1e-6 * np.max(np.abs(ref[3]))


# ------------------------------------------------------------------------------- multigrid
def aggregation_P(n, mask):
    """Piecewise-constant prolongation (DESIGN R-19): fine node c belongs to coarse node c' with
    c'_a = c_a // 2 on the coarsened axes (bit a of mask) and c'_a = c_a elsewhere."""
    dim = len(n)
    nc = tuple(v // 2 if (mask >> a) & 1 else v for a, v in enumerate(n))
    Nf, Nc = int(np.prod(n)), int(np.prod(nc))
    P = np.zeros((Nf, Nc))
    for f in range(Nf):
        c = np.unravel_index(f, tuple(reversed(n)))[::-1]            # (x, y, z)
        cc = [c[a] // 2 if (mask >> a) & 1 else c[a] for a in range(dim)]
        P[f, np.ravel_multi_index(tuple(reversed(cc)), tuple(reversed(nc)))] = 1.0
    return P, nc


@pytest.mark.parametrize("n,mask,beta", [((8, 6), 3, 0.0), ((8, 6), 1, 0.2), ((8, 6), 2, 0.0),
                                         ((4, 6, 4), 7, 0.1), ((4, 6, 4), 3, 0.0), ((4, 6, 4), 5, 0.0)])
def test_coarse_faces_are_galerkin_product(n, mask, beta):
    """The coarse operator assembled from the coarsened faces (coarse face = sum of the fine faces
    it covers, beta_c = 2^k beta) equals P^T A P exactly up to rounding; restrict = P^T,
    prolong = P.  Catches: pairing along the wrong numpy axis, a missing beta scale, summing the
    covered faces of the wrong parity."""
    F = rand_faces(n, 95)
    A = assemble_A(n, F, beta)
    P, nc = aggregation_P(n, mask)
    k = bin(mask).count("1")
    Ac = assemble_A(nc, coarsen_faces(F, n, mask), beta * 2 ** k)
    G = P.T @ A @ P
    assert np.max(np.abs(Ac - G)) <= 1e-13 * np.max(np.abs(G))
    r = gen.uniform(2, gen.STREAM_TEST, int(np.prod(n)))
    shape = tuple(reversed(n))
    assert np.max(np.abs(restrict(r.reshape(shape), mask).ravel() - P.T @ r)) <= 1e-14 * np.max(np.abs(P.T @ r))
    xc = gen.uniform(3, gen.STREAM_TEST, int(np.prod(nc)))
    assert np.array_equal(prolong(xc.reshape(tuple(reversed(nc))), mask).ravel(), P @ xc)


def dense_cycle(As, Ps, Sm, lev, r, sc, gamma):
    """x = B_lev r with dense matrices: S smoothing, P^T restriction, coarse cycle(s), s P
    correction, S post-smoothing."""
    if lev == len(As) - 1:
        return Sm[lev][1] @ r
    A, S = As[lev], Sm[lev][0]
    x = S @ r
    rc = Ps[lev].T @ (r - A @ x)
    xc = dense_cycle(As, Ps, Sm, lev + 1, rc, sc, gamma)
    if gamma == 2 and lev + 1 < len(As) - 1:
        xc = xc + dense_cycle(As, Ps, Sm, lev + 1, rc - As[lev + 1] @ xc, sc, gamma)
    x = x + sc * (Ps[lev] @ xc)
    return x + S @ (r - A @ x)


@pytest.mark.parametrize("n,tile,mask,nu,theta,gamma", [((16, 16), (8, 8), 3, 1, 0.5, 1),
                                                        ((16, 8), (8, 4), 1, 2, 0.6, 1),
                                                        ((16, 16), (8, 8), 3, 1, 0.45, 2),
                                                        ((8, 8, 4), (4, 4, 2), 3, 1, 0.5, 1)])
def test_vcycle_composition_matches_dense_cycle(n, tile, mask, nu, theta, gamma):
    """tests/mg_compose.vcycle (the expected value of the GPU multigrid tests) equals the cycle
    written with dense matrices: A_c = P^T A P, smoother S = theta M_m with M_1 = P_SGS^-1 and
    M_{j+1} = M_j + P_SGS^-1 (I - theta A M_j) (DESIGN R-17), coarsest level nu_c steps.
    Catches: restriction of r instead of r - A x, a missing coarse scale, pre- and post-smoothing
    from the wrong residual, the W-cycle's second coarse solve on the wrong right-hand side."""
    F = rand_faces(n, 97)
    levels, nu_c, sc = 3, 3, 1.3
    pbs = build_levels(n, tile, F, 0.0, levels, mask)
    As, Ps, Sm = [assemble_A(n, F, 0.0)], [], []
    nn = tuple(n)
    for _ in range(levels - 1):
        P, nc = aggregation_P(nn, mask)
        Ps.append(P)
        As.append(P.T @ As[-1] @ P)
        nn = nc
    for lev, pb in enumerate(pbs):
        N = pb.size
        Pinv = precond_inverse(lambda r: O.ssor_apply(pb, 1.0, r, 0), N, pb.shape)
        I = np.eye(N)

        def steps(m):
            M = Pinv.copy()
            for _ in range(m - 1):
                M = M + Pinv @ (I - theta * As[lev] @ M)
            return theta * M
        Sm.append((steps(nu), steps(nu_c)))
    r = gen.uniform(6, gen.STREAM_TEST, pbs[0].size)
    want = dense_cycle(As, Ps, Sm, 0, r, sc, gamma)
    got = vcycle(pbs, 0, r.reshape(pbs[0].shape), nu, theta, nu_c, sc, mask, gamma).ravel()
    assert np.max(np.abs(got - want)) <= 1e-12 * np.max(np.abs(want))
