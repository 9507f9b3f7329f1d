"""Oracle pins against closed forms, the paper's written coupled systems and dense
linear algebra (-m "not gpu").  Each test names what pins it."""
import numpy as np
import pytest

import oracle as O
from paper_1008_3699_b200 import gen


def rand_faces(n, seed, lo=0.5, hi=2.0):
    return tuple(lo + (hi - lo) * gen.unit(seed, gen.STREAM_TEST + a, int(np.prod(O.face_shape(n, a)))).reshape(
        O.face_shape(n, a)) for a in range(len(n)))


def sweep_matrix(pb, omega, phase, override=-1):
    """Iteration matrix of one sweep (b = 0), columns = images of unit vectors."""
    N = pb.size
    T = np.empty((N, N))
    z = np.zeros(pb.shape)
    for j in range(N):
        e = np.zeros(N)
        e[j] = 1.0
        T[:, j] = O.sweep(pb, omega, e.reshape(pb.shape), z, phase=phase, override=override).ravel()
    return T


def dense_A(pb):
    N = pb.size
    A = np.empty((N, N))
    for j in range(N):
        e = np.zeros(N)
        e[j] = 1.0
        A[:, j] = O.apply_A(pb, e.reshape(pb.shape)).ravel()
    return A


# ------------------------------------------------------------------ classical theory
def test_young_gs_and_sor_spectral_radius():
    """Model Poisson, lexicographic sweep (one box, fixed SW corner): rho(GS) = cos^2(pi h) and
    rho(SOR) = w - 1 for w >= w_opt = 2/(1+sin pi h) (Young; SURVEY §8(c) pin table)."""
    n = 7
    h = 1.0 / (n + 1)
    pb = O.tiled((n, n), (n, n))
    rho = max(abs(np.linalg.eigvals(sweep_matrix(pb, 1.0, 0, override=0))))
    assert abs(rho - np.cos(np.pi * h) ** 2) < 1e-10
    wopt = 2.0 / (1.0 + np.sin(np.pi * h))
    for w in (wopt + 0.05, 1.7):
        rho = max(abs(np.linalg.eigvals(sweep_matrix(pb, w, 0, override=0))))
        assert abs(rho - (w - 1.0)) < 1e-6
    # 1D: rho(GS) = cos^2(pi h)
    pb1 = O.tiled((15,), (15,))
    rho = max(abs(np.linalg.eigvals(sweep_matrix(pb1, 1.0, 0, override=0))))
    assert abs(rho - np.cos(np.pi / 16) ** 2) < 1e-10


def test_one_box_equals_classical_directional_sor():
    """p = 1: each decomposed sweep IS the classical directional sweep of its corner
    (PAPER:222-238, 493-522), here against the independent textbook loop nest."""
    rng = np.random.default_rng(0)
    for n in [(9,), (7, 6), (5, 4, 3)]:
        pb = O.tiled(n, n, faces=rand_faces(n, 3), beta=0.1)
        x = rng.standard_normal(pb.shape)
        b = rng.standard_normal(pb.shape)
        for corner in range(2 ** len(n)):
            for w in (0.7, 1.0, 1.6):
                got = O.sweep(pb, w, x, b, override=corner)
                ref = O.sor_lex(pb, w, x, b, corner)
                assert np.max(np.abs(got - ref)) <= 1e-13 * np.max(np.abs(ref))


def test_schedule_matches_paper_worked_example():
    """6x6 grid, 2x2 boxes: boxes 1..4 sweep NE, NW, SE, SW at iteration k and SW, SE, NW, NE at
    k+1.  Bits: bit0 = start at max x (E), bit1 = start at max y (N)."""
    pb = O.tiled((6, 6), (3, 3))
    names = {0: "SW", 1: "SE", 2: "NW", 3: "NE"}
    for phase, want in ((0, ["NE", "NW", "SE", "SW"]), (1, ["SW", "SE", "NW", "NE"])):
        bits, _ = O.node_info(pb, phase)
        got = [names[int(bits[y, x])] for (x, y) in ((0, 0), (3, 0), (0, 3), (3, 3))]
        assert got == want


def test_coupled_system_structure():
    """Coupled systems are the SCCs: 2D 6x6/2x2 boxes -> one 4x4 (12 nonzeros, eq 2d:sor4b4
    PAPER:578-630) and 2x2 edge pairs at phase 0, none at phase 1 ("no need to solution some local
    system"); 3D corner system 8x8 with 32 nonzeros."""
    s0 = O.scc_stats(O.tiled((6, 6), (3, 3)), 0)
    assert s0[4] == (1, 12) and s0[2][0] == 8
    assert set(O.scc_stats(O.tiled((6, 6), (3, 3)), 1)) == {1}
    s3 = O.scc_stats(O.tiled((6, 6, 6), (3, 3, 3)), 0)
    assert s3[8] == (1, 32)
    assert set(O.scc_stats(O.tiled((6, 6, 6), (3, 3, 3)), 1)) == {1}


def _fx(F, i, j):
    return F[0][j, i]


def test_paper_4x4_and_2x2_systems_2d():
    """Brute force against the systems the paper writes out: eq 2d:sor4b4 (with the
    row-2 denominator a^P_{i+1,j}) and eq 2d:sor2b2 (with f added and u_{i-1,j+1}^(k)
    in row 2), on a 6x6 grid with 2x2 boxes and a distinct omega per direction."""
    n = (6, 6)
    F = rand_faces(n, 11)
    pb = O.Problem(n, (O.uniform_bounds(6, 3), O.uniform_bounds(6, 3)), F, 0.0)
    rng = np.random.default_rng(5)
    u = rng.standard_normal(pb.shape)          # u[y, x]
    f = rng.standard_normal(pb.shape)
    om = np.array([1.1, 1.3, 0.9, 1.45])       # index = direction bits: SW, SE, NW, NE
    wSW, wSE, wNW, wNE = om
    new = O.sweep(pb, om, u, f, phase=0)

    def aE(i, j): return F[0][j, i + 1]
    def aW(i, j): return F[0][j, i]
    def aN(i, j): return F[1][j + 1, i]
    def aS(i, j): return F[1][j, i]
    def aP(i, j): return aE(i, j) + aW(i, j) + aN(i, j) + aS(i, j)
    def U(i, j): return u[j, i]
    def Fr(i, j): return f[j, i]

    i, j = 2, 2                                # node #1 of Omega_1 (0-based)
    M = np.array([
        [1, -wNE * aE(i, j) / aP(i, j), -wNE * aN(i, j) / aP(i, j), 0],
        [-wNW * aW(i + 1, j) / aP(i + 1, j), 1, 0, -wNW * aN(i + 1, j) / aP(i + 1, j)],
        [-wSE * aS(i, j + 1) / aP(i, j + 1), 0, 1, -wSE * aE(i, j + 1) / aP(i, j + 1)],
        [0, -wSW * aS(i + 1, j + 1) / aP(i + 1, j + 1), -wSW * aW(i + 1, j + 1) / aP(i + 1, j + 1), 1]])
    r = np.array([
        (1 - wNE) * U(i, j) + wNE * (aS(i, j) * U(i, j - 1) + aW(i, j) * U(i - 1, j) + Fr(i, j)) / aP(i, j),
        (1 - wNW) * U(i + 1, j) + wNW * (aS(i + 1, j) * U(i + 1, j - 1) + aE(i + 1, j) * U(i + 2, j)
                                         + Fr(i + 1, j)) / aP(i + 1, j),
        (1 - wSE) * U(i, j + 1) + wSE * (aW(i, j + 1) * U(i - 1, j + 1) + aN(i, j + 1) * U(i, j + 2)
                                         + Fr(i, j + 1)) / aP(i, j + 1),
        (1 - wSW) * U(i + 1, j + 1) + wSW * (aE(i + 1, j + 1) * U(i + 2, j + 1) + aN(i + 1, j + 1) * U(i + 1, j + 2)
                                             + Fr(i + 1, j + 1)) / aP(i + 1, j + 1)])
    sol = np.linalg.solve(M, r)
    got = np.array([new[j, i], new[j, i + 1], new[j + 1, i], new[j + 1, i + 1]])
    assert np.max(np.abs(got - sol)) < 1e-14 * np.max(np.abs(sol)) * 10
    # eq 2d:sor2b2: nodes (i-1, j) in Omega_1 (NE) and (i-1, j+1) in Omega_3 (SE)
    ui_j, ui_j1 = new[j, i], new[j + 1, i]
    M2 = np.array([[1, -wNE * aN(i - 1, j) / aP(i - 1, j)],
                   [-wSE * aS(i - 1, j + 1) / aP(i - 1, j + 1), 1]])
    r2 = np.array([
        (1 - wNE) * U(i - 1, j) + wNE * (aS(i - 1, j) * U(i - 1, j - 1) + aW(i - 1, j) * U(i - 2, j)
                                         + aE(i - 1, j) * ui_j + Fr(i - 1, j)) / aP(i - 1, j),
        (1 - wSE) * U(i - 1, j + 1) + wSE * (aW(i - 1, j + 1) * U(i - 2, j + 1) + aE(i - 1, j + 1) * ui_j1
                                             + aN(i - 1, j + 1) * U(i - 1, j + 2) + Fr(i - 1, j + 1)) / aP(i - 1, j + 1)])
    sol2 = np.linalg.solve(M2, r2)
    got2 = np.array([new[j, i - 1], new[j + 1, i - 1]])
    assert np.max(np.abs(got2 - sol2)) < 1e-13 * np.max(np.abs(sol2))


def test_paper_2x2_system_1d():
    """eq 1d:sorc: two boxes, second iteration (box 1 RL, box 2 LR) couples x_m and
    x_{m+1}; distinct w_L, w_R; a_i, c_i from random faces."""
    n = (10,)
    F = rand_faces(n, 21)
    pb = O.Problem(n, (np.array([0, 5, 10]),), F, 0.0)
    rng = np.random.default_rng(2)
    u = rng.standard_normal(10)
    f = rng.standard_normal(10)
    wL, wR = 1.3, 0.8
    new = O.sweep(pb, [wL, wR], u, f, phase=1)
    a = F[0][1:]          # a_i: face between i and i+1
    c = F[0][:-1]         # c_i: face between i-1 and i
    b = a + c
    m = 4
    M = np.array([[1, -a[m] * wR / b[m]], [-c[m + 1] * wL / b[m + 1], 1]])
    r = np.array([(1 - wR) * u[m] + wR / b[m] * (c[m] * u[m - 1] + f[m]),
                  (1 - wL) * u[m + 1] + wL / b[m + 1] * (a[m + 1] * u[m + 2] + f[m + 1])])
    sol = np.linalg.solve(M, r)
    assert np.max(np.abs(new[m:m + 2] - sol)) < 1e-14 * np.max(np.abs(sol)) * 10
    # first iteration (box 1 LR from the left boundary, box 2 RL from the right): no coupling,
    # each box is an independent directional sweep with old neighbour values
    new0 = O.sweep(pb, [wL, wR], u, f, phase=0)
    ref = u.copy()
    for i in range(5):
        ref[i] = (1 - wL) * u[i] + wL / b[i] * (c[i] * (ref[i - 1] if i > 0 else 0) + a[i] * u[i + 1] + f[i])
    for i in range(9, 4, -1):
        ref[i] = (1 - wR) * u[i] + wR / b[i] * (c[i] * u[i - 1] + a[i] * (ref[i + 1] if i < 9 else 0) + f[i])
    assert np.max(np.abs(new0 - ref)) < 1e-14 * np.max(np.abs(ref)) * 10


@pytest.mark.parametrize("n,tile", [((8, 8), (4, 4)), ((12, 10), (4, 5)), ((6, 6, 6), (3, 3, 3)), ((4, 6, 4), (2, 3, 2))])
def test_per_node_equations_hold(n, tile):
    """Every node of the output satisfies its own directional update formula (eqs sor2d_sw..nw,
    PAPER:493-522, 3D analogue PAPER:868-895): implicit (start-side) neighbours at the new values,
    the others at the old values; i.e. the coupled solves are exact."""
    F = rand_faces(n, 31)
    pb = O.tiled(n, tile, faces=F, beta=0.05)
    rng = np.random.default_rng(7)
    u = rng.standard_normal(pb.shape)
    f = rng.standard_normal(pb.shape)
    dim = len(n)
    om = 0.6 + 0.1 * np.arange(2 ** dim)
    for phase in range(2 ** dim):
        new = O.sweep(pb, om, u, f, phase=phase)
        bits, _ = O.node_info(pb, phase)
        worst = 0.0
        for idx in np.ndindex(*pb.shape):
            c = idx[::-1]                       # (x, y, z)
            s = int(bits[idx])
            w = om[s]
            acc = f[idx]
            ap = pb.beta
            for a in range(dim):
                for sd in (-1, 1):
                    q = list(c)
                    q[a] += sd
                    fi = [c[t] for t in range(dim)]
                    if sd > 0:
                        fi[a] += 1
                    coef = F[a][tuple(fi[::-1])]
                    ap += coef
                    if not (0 <= q[a] < n[a]):
                        continue
                    implicit = (sd == (1 if (s >> a) & 1 else -1))
                    acc += coef * (new if implicit else u)[tuple(q[::-1])]
            val = (1 - w) * u[idx] + w / ap * acc
            worst = max(worst, abs(val - new[idx]))
        assert worst < 1e-13


def test_manufactured_solution_converges_exactly():
    """u = prod x_i on the boundary is reproduced exactly by the discrete solution:
    the decomposed sweep (4x4 boxes, w = 1.5) converges to it to round-off."""
    from oracle.model import model_problem
    for dim, R, parts, nsw in ((2, 18, [4, 4], 400), (3, 10, [2, 2, 2], 200)):
        pb, b, exact = model_problem(dim, R, parts)
        u = np.zeros(pb.shape)
        for k in range(nsw):
            u = O.sweep(pb, 1.5, u, b, phase=k)
        assert np.max(np.abs(u - exact)) < 1e-12


def test_discretisation_error_second_order():
    """u = sin(pi x) sin(pi y): the converged discrete solution's error drops ~4x per h-halving."""
    errs = []
    for n in (15, 31):
        h = 1.0 / (n + 1)
        xs = np.arange(1, n + 1) * h
        X, Y = np.meshgrid(xs, xs, indexing="xy")
        ue = np.sin(np.pi * X) * np.sin(np.pi * Y)
        f = 2 * np.pi ** 2 * ue * h * h
        pb = O.tiled((n, n), (n, n))
        x, it, rr, ok = O.pcg(pb, f, precond=0, rtol=1e-13, maxit=5000)
        assert ok
        errs.append(np.max(np.abs(x - ue)))
    assert 3.6 < errs[0] / errs[1] < 4.4


def test_decomposed_spectral_radius_below_one_and_close_to_sequential():
    """rho(T_cycle) < 1 for random (boxes, omega) on Poisson 8x8 (PAPER:1059-1192 conclusion; the
    paper's bound itself is false, R-16) and close to the one-box same-schedule value
    ("number of iterations ... close to that of sequential")."""
    rng = np.random.default_rng(3)
    seq_cache = {}
    for trial in range(6):
        w = float(rng.uniform(0.4, 1.9))
        tx, ty = [(2, 2), (4, 4), (2, 4), (4, 2), (8, 4), (4, 8)][trial]
        pb = O.tiled((8, 8), (tx, ty))
        T = np.eye(64)
        for k in range(4):
            T = sweep_matrix(pb, w, k) @ T
        rho = max(abs(np.linalg.eigvals(T)))
        assert rho < 1.0
        pb1 = O.tiled((8, 8), (8, 8))
        T1 = np.eye(64)
        for k in range(4):
            T1 = sweep_matrix(pb1, w, k) @ T1
        rho1 = max(abs(np.linalg.eigvals(T1)))
        assert abs(rho - rho1) < 0.08, (w, tx, ty, rho, rho1)


def test_tile_locality_width_two():
    """GPU design premise (SURVEY §8(c) tile locality): a box's new values depend only on old values
    within two layers of the box; one layer is NOT enough when the box has a coupled start face."""
    n, t = (12, 12), (4, 4)
    pb = O.tiled(n, t, faces=rand_faces(n, 41))
    rng = np.random.default_rng(9)
    u = rng.standard_normal(pb.shape)
    f = rng.standard_normal(pb.shape)
    for phase in range(4):
        base = O.sweep(pb, 1.2, u, f, phase=phase)
        for bx, by in ((1, 1), (0, 1), (2, 2)):
            x0, y0 = 4 * bx, 4 * by
            for width, must_hold in ((2, True), (1, False)):
                v = u.copy()
                mask = np.ones(pb.shape, bool)
                mask[max(0, y0 - width):y0 + 4 + width, max(0, x0 - width):x0 + 4 + width] = False
                v[mask] += 10.0
                got = O.sweep(pb, 1.2, v, f, phase=phase)
                same = np.array_equal(got[y0:y0 + 4, x0:x0 + 4], base[y0:y0 + 4, x0:x0 + 4])
                if must_hold:
                    assert same
                elif phase == 0 and (bx, by) == (1, 1):
                    assert not same


# ------------------------------------------------------------------ ILU / SSOR / PCG
def textbook_ilu0(A):
    """Saad Algorithm 10.4 (IKJ ILU(0)) on a dense matrix restricted to A's pattern."""
    N = A.shape[0]
    LU = A.copy()
    pat = A != 0
    for i in range(1, N):
        for k in range(i):
            if not pat[i, k]:
                continue
            LU[i, k] /= LU[k, k]
            for j in range(k + 1, N):
                if pat[i, j]:
                    LU[i, j] -= LU[i, k] * LU[k, j]
    L = np.tril(LU, -1) + np.eye(N)
    U = np.triu(LU)
    return L, U


def precond_matrix(apply, N, shape):
    Pinv = np.empty((N, N))
    for j in range(N):
        e = np.zeros(N)
        e[j] = 1.0
        Pinv[:, j] = apply(e.reshape(shape)).ravel()
    return np.linalg.inv(Pinv)


@pytest.mark.parametrize("n", [(9,), (5, 6), (3, 4, 3)])
def test_one_box_ilu0_is_classical_ilu0(n):
    """One box, natural (SW) ordering: the D~-recurrence ILU(0) equals textbook ILU(0) (Saad Alg. 10.4,
    the reference PAPER:916-921 cites) in both pairings; 1D ILU(0) = exact LU (P = A)."""
    F = rand_faces(n, 51)
    pb = O.tiled(n, n, faces=F, beta=0.0)
    A = dense_A(pb)
    L, U = textbook_ilu0(A)
    invD = O.ilu0_factor(pb, override=0)
    for pairing in (0, 1):
        P = precond_matrix(lambda r: O.ilu_apply(pb, invD, r, pairing, override=0), pb.size, pb.shape)
        assert np.max(np.abs(P - L @ U)) < 1e-12 * np.max(np.abs(A))
    if len(n) == 1:
        P = precond_matrix(lambda r: O.ilu_apply(pb, invD, r, 0, override=0), pb.size, pb.shape)
        assert np.max(np.abs(P - A)) < 1e-12 * np.max(np.abs(A))


@pytest.mark.parametrize("n,tile", [((8, 8), (4, 4)), ((12, 10), (4, 5)), ((6, 6, 6), (3, 3, 3))])
def test_decomposed_ilu_properties(n, tile):
    """PAPER pairing: (D~+L) D~^-1 (D~+U) = A on A's sparsity pattern (an exact ILU(0) of the
    alternating block-triangular splitting).  SYMMETRIC pairing: P = P^T,
    positive definite."""
    F = rand_faces(n, 61)
    pb = O.tiled(n, tile, faces=F, beta=0.0)
    A = dense_A(pb)
    invD = O.ilu0_factor(pb, phase=0)
    P1 = precond_matrix(lambda r: O.ilu_apply(pb, invD, r, 1), pb.size, pb.shape)
    pat = A != 0
    assert np.max(np.abs((P1 - A)[pat])) < 1e-12 * np.max(np.abs(A))
    P0 = precond_matrix(lambda r: O.ilu_apply(pb, invD, r, 0), pb.size, pb.shape)
    assert np.max(np.abs(P0 - P0.T)) < 1e-12 * np.max(np.abs(A))
    assert np.min(np.linalg.eigvalsh(0.5 * (P0 + P0.T))) > 0


def test_one_box_ssor_is_textbook_ssor():
    """SSOR preconditioner with one box, SW ordering:
    M = (D/w + L) (w/(2-w)) D^-1 (D/w + U)."""
    n = (5, 6)
    pb = O.tiled(n, n, faces=rand_faces(n, 71), beta=0.2)
    A = dense_A(pb)
    D = np.diag(np.diag(A))
    L = np.tril(A, -1)
    U = np.triu(A, 1)
    for w in (1.0, 1.4):
        M = (D / w + L) @ (w / (2 - w) * np.linalg.inv(D)) @ (D / w + U)
        for pairing in (0, 1):
            P = precond_matrix(lambda r: O.ssor_apply(pb, w, r, pairing, override=0), pb.size, pb.shape)
            assert np.max(np.abs(P - M)) < 1e-11 * np.max(np.abs(M))


def test_pcg_against_textbook_cg_and_direct_solve():
    """No preconditioner = textbook CG (same iterates); preconditioned solves reach the direct
    solution; 1D one-box ILU(0) is exact, so PCG converges in one iteration."""
    n = (12, 10)
    F = rand_faces(n, 81)
    pb = O.tiled(n, (4, 5), faces=F, beta=0.0)
    A = dense_A(pb)
    b = gen.uniform(0, gen.STREAM_RHS, pb.size)
    xd = np.linalg.solve(A, b)
    # textbook CG
    x = np.zeros_like(b)
    r = b.copy()
    p = r.copy()
    rr = r @ r
    it_ref = None
    for it in range(1, 500):
        q = A @ p
        al = rr / (p @ q)
        x += al * p
        r -= al * q
        rrn = r @ r
        if np.sqrt(rrn) / np.linalg.norm(b) < 1e-10:
            it_ref = it
            break
        p = r + rrn / rr * p
        rr = rrn
    xo, it, rel, ok = O.pcg(pb, b, precond=0, rtol=1e-10)
    assert ok and abs(it - it_ref) <= 1
    cond_tol = 1e-10 * np.linalg.cond(A)
    assert np.linalg.norm(xo.ravel() - xd) / np.linalg.norm(xd) < cond_tol
    for pc, w in ((1, 1.0), (2, 1.0)):
        xo, it2, rel, ok = O.pcg(pb, b, precond=pc, omega=w, pairing=0, rtol=1e-10)
        assert ok and it2 < it
        assert np.linalg.norm(xo.ravel() - xd) / np.linalg.norm(xd) < cond_tol
    # flexible PCG with the nonsymmetric PAPER pairing still converges
    xo, it3, rel, ok = O.pcg(pb, b, precond=2, pairing=1, flexible=True, rtol=1e-10)
    assert ok
    pb1 = O.tiled((20,), (20,), faces=rand_faces((20,), 3))
    b1 = gen.uniform(0, gen.STREAM_RHS, 20)
    xo, it, rel, ok = O.pcg(pb1, b1, precond=2, override=0, rtol=1e-12)
    assert ok and it == 1


def test_faces_from_k_harmonic_mean():
    """Harmonic face mean: k = 2, 4 -> 8/3 (SPEC example); constant k
    gives the per-axis scale exactly; symmetric in its arguments."""
    k = np.array([2.0, 4.0, 4.0])
    f = O.faces_from_k((1,), k)[0]
    assert abs(f[0] - 8.0 / 3.0) < 1e-15 and f[1] == 4.0
    kk = np.full((5, 6, 7), 3.0)
    F = O.faces_from_k((5, 4, 3), kk, scale=(1.0, 0.1, 0.01))
    assert np.all(F[0] == 3.0) and np.all(F[1] == 0.1 * 3.0) and np.all(F[2] == 0.01 * 3.0)
    kr = np.exp(gen.normal_field(0, gen.STREAM_LOGK, (6, 7)))
    F = O.faces_from_k((5, 4), kr)
    Fr = O.faces_from_k((5, 4), kr[::-1, ::-1].copy())
    assert np.allclose(F[0], Fr[0][::-1, ::-1], rtol=0, atol=0)


def test_decomposed_symmetric_preconditioner_spectrum_reaches_two():
    """The decomposed SGS / D-ILU(0) preconditioners of the SYMMETRIC pairing (reading R-C) have
    lambda(P^-1 A) in (0, 2] with the maximum 2 attained (the start-face pairs), while the
    one-box (classical) SGS has lambda_max = 1.  Hence the m-step form z_{j+1} = z_j +
    P^-1 (r - theta A z_j) of sw_set_precond_steps needs theta < 1 for even m (include/sweep.h)."""
    import numpy as np
    n = (24, 24)
    N = n[0] * n[1]

    def spectrum(tile, ilu):
        pb = O.tiled(n, tile)
        inv = O.ilu0_factor(pb) if ilu else None
        Pi = np.zeros((N, N))
        A = np.zeros((N, N))
        for i in range(N):
            e = np.zeros(N)
            e[i] = 1.0
            e = e.reshape(pb.shape)
            Pi[:, i] = (O.ilu_apply(pb, inv, e, 0) if ilu else O.ssor_apply(pb, 1.0, e, 0)).ravel()
            A[:, i] = O.apply_A(pb, e).ravel()
        ev = np.linalg.eigvals(Pi @ A)
        assert np.max(np.abs(ev.imag)) < 1e-8
        return ev.real.min(), ev.real.max()
    lo, hi = spectrum((8, 8), False)
    assert lo > 0 and abs(hi - 2.0) < 1e-9
    lo, hi = spectrum((8, 8), True)
    assert lo > 0 and abs(hi - 2.0) < 1e-9
    lo, hi = spectrum(n, False)
    assert lo > 0 and abs(hi - 1.0) < 1e-9
