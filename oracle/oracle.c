/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, single-threaded CPU oracle for the decomposed multi-frontal SOR /
 * SSOR / ILU(0) sweeps of arXiv 1008.3699 (Tavakoli, "Parallelizing sequential
 * sweeping on structured grids").  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.  It
 * shares no code with the CUDA path (paper_1008_3699_b200/csrc).
 *
 * Citations "PAPER:n" are line numbers of /root/reference/PAPER.md; "SURVEY §x" is
 * /root/repo/SURVEY.md; readings "R-n" are listed in DESIGN.md §3.
 *
 * Layout: interior nodes only, x fastest: idx = i + n0*(j + n1*k).  Axes that a
 * lower-dimensional problem does not use have n = 1.  Face coefficient arrays:
 * face[a] has shape n with n_a+1 along axis a; face[a][c] is the coefficient of
 * the face between node c - e_a and node c (c_a in 0..n_a).  face[a] == NULL
 * means every face coefficient of that axis is 1.0 (Poisson, h^2-scaled).
 * Dirichlet boundary values are folded into b, so every node
 * outside the domain has value 0 and its term is OMITTED below.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_ESINGULAR 2
#define OR_ENOCONV 3
#define OR_EORDER 4   /* dependency order violated: the method would not be a triangular solve */
#define OR_ENOMEM 5
#define OR_EINVAL 6

typedef struct {
    int dim;                  /* 1, 2 or 3 */
    int64_t n[3];             /* interior nodes per axis (1 for unused axes) */
    const double *face[3];    /* NULL = all ones */
    double beta;              /* reaction coefficient (a_P = sum faces + beta) */
    int nbox[3];              /* boxes per axis */
    const int64_t *bounds[3]; /* bounds[a][0..nbox[a]]: box r along a is [bounds[r], bounds[r+1]) */
} or_grid;

/* ------------------------------------------------------------------ geometry */

static int64_t n_nodes(const or_grid *g) { return g->n[0] * g->n[1] * g->n[2]; }

static void coords_of(const or_grid *g, int64_t idx, int64_t c[3]) {
    c[0] = idx % g->n[0];
    int64_t t = idx / g->n[0];
    c[1] = t % g->n[1];
    c[2] = t / g->n[1];
}

static int64_t lin(const or_grid *g, const int64_t c[3]) { return c[0] + g->n[0] * (c[1] + g->n[1] * c[2]); }

static int inside(const or_grid *g, const int64_t c[3]) {
    for (int a = 0; a < 3; ++a)
        if (c[a] < 0 || c[a] >= g->n[a]) return 0;
    return 1;
}

/* coefficient of the face between c - e_a and c (c[a] may equal n_a) */
static double face_minus(const or_grid *g, const int64_t c[3], int a) {
    if (!g->face[a]) return 1.0;
    int64_t m0 = g->n[0] + (a == 0), m1 = g->n[1] + (a == 1);
    return g->face[a][c[0] + m0 * (c[1] + m1 * c[2])];
}

/* coefficient c_ij of the face between node c and its neighbour c + sd*e_a */
static double face_between(const or_grid *g, const int64_t c[3], int a, int sd) {
    int64_t f[3] = {c[0], c[1], c[2]};
    if (sd > 0) f[a] += 1;
    return face_minus(g, f, a);
}

/* a_P = a^W + a^E + a^S + a^N (+ a^B + a^F) + beta, PAPER:429-430 (2D), 192 (1D);
 * summed per axis pair first, a_P = ((F_x- + F_x+) + (F_y- + F_y+)) + (F_z- + F_z+), then
 * beta (reading R-7).  Each pair sum is commutative, so the value does not depend on the
 * direction a box is swept in. */
static double a_p(const or_grid *g, const int64_t c[3]) {
    double s = 0.0;
    for (int a = 0; a < g->dim; ++a) {
        double pair = face_between(g, c, a, -1) + face_between(g, c, a, +1);
        s = (a == 0) ? pair : s + pair;
    }
    return s + g->beta;
}

/* ---------------------------------------------------------------- schedule
 * Sweep-direction rules of PAPER:781-807 (2D) and PAPER:868-878 (3D); 1D rule
 * PAPER:335-338.  A box's start side along axis a is s_a = c_a(k mod 2^d) XOR
 * (r_a mod 2), s_a = 1 meaning "starts at the max end" (reading R-4, R-5):
 *   1D  c = [0 (LR), 1 (RL)]                    -- odd boxes LR first
 *   2D  c = [NE, SW, NW, SE]                     -- box 1 sweeps NE first
 *   3D  8 corners, pairs are full reversals, each pair a new diagonal
 * ov >= 0 replaces c(k) by the fixed corner ov (classical directional sweeps).
 */
static const int CYC1[2] = {0, 1};
static const int CYC2[4] = {3, 0, 2, 1};                 /* bits (sx | sy<<1): NE, SW, NW, SE */
static const int CYC3[8] = {7, 0, 6, 1, 5, 2, 3, 4};     /* (1,1,1),(0,0,0),(0,1,1),(1,0,0),(1,0,1),(0,1,0),(1,1,0),(0,0,1) */

int or_base_bits(int dim, int64_t phase, int ov) {
    if (ov >= 0) return ov;
    int64_t m = (int64_t)1 << dim;
    int64_t k = ((phase % m) + m) % m;
    if (dim == 1) return CYC1[k];
    if (dim == 2) return CYC2[k];
    return CYC3[k];
}

/* per-run tables: box index of every coordinate along every axis */
typedef struct {
    const or_grid *g;
    int *boxof[3];
    int base;          /* c(k) bits */
} ctx_t;

static int ctx_init(ctx_t *x, const or_grid *g, int64_t phase, int ov) {
    memset(x, 0, sizeof(*x));
    x->g = g;
    x->base = or_base_bits(g->dim, phase, ov);
    for (int a = 0; a < 3; ++a) {
        x->boxof[a] = (int *)malloc(sizeof(int) * (size_t)g->n[a]);
        if (!x->boxof[a]) return OR_ENOMEM;
        if (a >= g->dim) {
            for (int64_t i = 0; i < g->n[a]; ++i) x->boxof[a][i] = 0;
            continue;
        }
        if (g->bounds[a][0] != 0 || g->bounds[a][g->nbox[a]] != g->n[a]) return OR_EINVAL;
        for (int r = 0; r < g->nbox[a]; ++r) {
            if (g->bounds[a][r + 1] <= g->bounds[a][r]) return OR_EINVAL;
            for (int64_t i = g->bounds[a][r]; i < g->bounds[a][r + 1]; ++i) x->boxof[a][i] = r;
        }
    }
    return OR_OK;
}

static void ctx_free(ctx_t *x) {
    for (int a = 0; a < 3; ++a) free(x->boxof[a]);
}

/* start side of node c's box along axis a (1 = starts at max end) */
static int start_bit(const ctx_t *x, const int64_t c[3], int a) {
    return ((x->base >> a) & 1) ^ (x->boxof[a][c[a]] & 1);
}

static int dir_bits(const ctx_t *x, const int64_t c[3]) {
    int s = 0;
    for (int a = 0; a < x->g->dim; ++a) s |= start_bit(x, c, a) << a;
    return s;
}

/* wavefront index: distance from the box's start corner (SPEC frontal order) */
static int64_t wave_d(const ctx_t *x, const int64_t c[3]) {
    const or_grid *g = x->g;
    int64_t d = 0;
    for (int a = 0; a < g->dim; ++a) {
        int r = x->boxof[a][c[a]];
        int64_t lo = g->bounds[a][r], hi = g->bounds[a][r + 1];
        d += start_bit(x, c, a) ? (hi - 1 - c[a]) : (c[a] - lo);
    }
    return d;
}

static int same_box(const ctx_t *x, const int64_t p[3], const int64_t q[3]) {
    for (int a = 0; a < x->g->dim; ++a)
        if (x->boxof[a][p[a]] != x->boxof[a][q[a]]) return 0;
    return 1;
}

/* "implicit" neighbour (PAPER:493-522 superscript (k+1) terms): neighbour q of p along
 * axis a on side sd is implicit for p iff q lies on the start side of p's box. */
static int is_implicit(const ctx_t *x, const int64_t p[3], int a, int sd) {
    return sd == (start_bit(x, p, a) ? +1 : -1);
}

/* dependency used by the triangular solves:
 *   forward  : p depends on q iff q is implicit for p           (matrix D/w + A_I)
 *   transpose: p depends on q iff p is implicit for q           (matrix D/w + A_I^T) */
static int depends(const ctx_t *x, int transpose, const int64_t p[3], int a, int sd) {
    if (!transpose) return is_implicit(x, p, a, sd);
    int64_t q[3] = {p[0], p[1], p[2]};
    q[a] += sd;
    return is_implicit(x, q, a, -sd);
}

/* ------------------------------------------------ coupled-system elimination
 * The paper's coupled 2x2 / 4x4 / 8x8 systems (eq 1d:sorc PAPER:289-304, eq 2d:sor4b4
 * PAPER:578-630, eq 2d:sor2b2 PAPER:642-673, 3D PAPER:884-893) "can be easily inverted"
 * (PAPER:305, 632).  Reading R-8: Gaussian elimination without pivoting in member
 * order (ascending global index), reciprocal pivots, fused multiply-adds. */
static int ge_solve(int k, double M[8][8], double *rhs, double *u, double *minpiv) {
    double inv[8];
    for (int p = 0; p < k; ++p) {
        double piv = M[p][p];
        if (minpiv && fabs(piv) < *minpiv) *minpiv = fabs(piv);
        if (!(fabs(piv) >= 1e-14)) return OR_ESINGULAR;
        inv[p] = 1.0 / piv;
        for (int q = p + 1; q < k; ++q) {
            double l = M[q][p] * inv[p];
            for (int j = p + 1; j < k; ++j) M[q][j] = fma(-l, M[p][j], M[q][j]);
            rhs[q] = fma(-l, rhs[p], rhs[q]);
        }
    }
    for (int p = k - 1; p >= 0; --p) {
        double s = rhs[p];
        for (int j = p + 1; j < k; ++j) s = fma(-M[p][j], u[j], s);
        u[p] = s * inv[p];
    }
    return OR_OK;
}

/* ----------------------------------------------------------- triangular solve
 * Solves, for every node p,
 *     out_p = r0_p + sum_{q in dep(p)} (alpha_p * c_pq) * out_q
 * i.e. the block-triangular system (I - diag(alpha) A_I) out = r0 (forward) or its
 * transpose-pattern analogue.  For the SOR sweep this is exactly the paper's update
 * formulas with the coupled systems of PAPER:289-304,
 * 578-680, 884-895 appearing as the strongly connected components (SCCs) of the
 * dependency graph.  Nodes are processed by wavefront index d
 * (ascending forward, descending transpose); every dependency outside the SCC must
 * already be final, which is CHECKED (OR_EORDER) rather than assumed. */
static int trisolve(const or_grid *g, int64_t phase, int ov, int transpose, const double *alpha,
                    const double *r0, double *out, double *minpiv) {
    ctx_t x;
    int st = ctx_init(&x, g, phase, ov);
    int64_t N = n_nodes(g);
    int64_t *dval = NULL, *order = NULL, *cnt = NULL;
    unsigned char *done = NULL;
    if (st != OR_OK) goto out;
    dval = (int64_t *)malloc(sizeof(int64_t) * (size_t)N);
    order = (int64_t *)malloc(sizeof(int64_t) * (size_t)N);
    done = (unsigned char *)calloc((size_t)N, 1);
    if (!dval || !order || !done) { st = OR_ENOMEM; goto out; }
    int64_t dmax = 0;
    for (int64_t i = 0; i < N; ++i) {
        int64_t c[3];
        coords_of(g, i, c);
        dval[i] = wave_d(&x, c);
        if (dval[i] > dmax) dmax = dval[i];
    }
    cnt = (int64_t *)calloc((size_t)(dmax + 2), sizeof(int64_t));
    if (!cnt) { st = OR_ENOMEM; goto out; }
    for (int64_t i = 0; i < N; ++i) cnt[dval[i] + 1]++;
    for (int64_t d = 0; d <= dmax; ++d) cnt[d + 1] += cnt[d];
    for (int64_t i = 0; i < N; ++i) order[cnt[dval[i]]++] = i;   /* stable: ascending index within d */

    for (int64_t t = 0; t < N; ++t) {
        int64_t i = transpose ? order[N - 1 - t] : order[t];
        if (done[i]) continue;
        /* SCC of i: closure under mutual dependencies */
        int64_t mem[8];
        int k = 1;
        mem[0] = i;
        for (int h = 0; h < k; ++h) {
            int64_t p[3];
            coords_of(g, mem[h], p);
            for (int a = 0; a < g->dim; ++a)
                for (int sd = -1; sd <= 1; sd += 2) {
                    int64_t q[3] = {p[0], p[1], p[2]};
                    q[a] += sd;
                    if (!inside(g, q)) continue;
                    if (depends(&x, transpose, p, a, sd) && depends(&x, transpose, q, a, -sd)) {
                        int64_t qi = lin(g, q);
                        int seen = 0;
                        for (int m = 0; m < k; ++m) seen |= (mem[m] == qi);
                        if (!seen) {
                            if (k == 8) { st = OR_EORDER; goto out; }
                            mem[k++] = qi;
                        }
                    }
                }
        }
        /* member order: ascending global index */
        for (int a1 = 1; a1 < k; ++a1)
            for (int b1 = a1; b1 > 0 && mem[b1 - 1] > mem[b1]; --b1) {
                int64_t tmp = mem[b1]; mem[b1] = mem[b1 - 1]; mem[b1 - 1] = tmp;
            }
        double M[8][8], rhs[8], u[8];
        for (int p = 0; p < k; ++p) {
            int64_t pc[3];
            coords_of(g, mem[p], pc);
            for (int q = 0; q < k; ++q) M[p][q] = (p == q) ? 1.0 : 0.0;
            double acc = r0[mem[p]];
            for (int a = 0; a < g->dim; ++a)
                for (int sd = -1; sd <= 1; sd += 2) {
                    int64_t qc[3] = {pc[0], pc[1], pc[2]};
                    qc[a] += sd;
                    if (!inside(g, qc) || !depends(&x, transpose, pc, a, sd)) continue;
                    int64_t qi = lin(g, qc);
                    double m = alpha[mem[p]] * face_between(g, pc, a, sd);
                    int inscc = -1;
                    for (int q = 0; q < k; ++q)
                        if (mem[q] == qi) inscc = q;
                    if (inscc >= 0) {
                        M[p][inscc] = -m;
                    } else {
                        if (!done[qi]) { st = OR_EORDER; goto out; }
                        acc = fma(m, out[qi], acc);
                    }
                }
            rhs[p] = acc;
        }
        if (k == 1) {
            u[0] = rhs[0];
        } else {
            st = ge_solve(k, M, rhs, u, minpiv);
            if (st != OR_OK) goto out;
        }
        for (int p = 0; p < k; ++p) {
            out[mem[p]] = u[p];
            done[mem[p]] = 1;
        }
    }
out:
    free(dval); free(order); free(done); free(cnt);
    ctx_free(&x);
    return st;
}

/* ------------------------------------------------------------ public: sweep
 * One decomposed SOR sweep at phase k (PAPER:326-346 1D, 524-693 2D, 860-895 3D):
 *   u+ = (D Omega^-1 + A_I(k))^-1 [ b + (D Omega^-1 - D) u - A_E(k) u ]
 * per-node rhs (reading R-7):
 *   alpha = w / a_P;  e = b + sum_{explicit q, axis order} c_pq u_q  (fma chain)
 *   r0 = fma(alpha, e, (1 - w) * u_p)
 * omega[] is indexed by the box's direction bits (bit a = s_a); n_omega == 1 uses omega[0]. */
int or_sweep(const or_grid *g, const double *omega, int n_omega, int64_t phase, int ov,
             const double *xold, const double *b, double *xnew, double *minpiv) {
    ctx_t x;
    int st = ctx_init(&x, g, phase, ov);
    int64_t N = n_nodes(g);
    double *alpha = (double *)malloc(sizeof(double) * (size_t)N);
    double *r0 = (double *)malloc(sizeof(double) * (size_t)N);
    if (st == OR_OK && (!alpha || !r0)) st = OR_ENOMEM;
    if (st == OR_OK) {
        for (int64_t i = 0; i < N; ++i) {
            int64_t c[3];
            coords_of(g, i, c);
            int s = dir_bits(&x, c);
            double w = omega[n_omega == 1 ? 0 : s];
            double al = w / a_p(g, c);
            double e = b[i];
            for (int a = 0; a < g->dim; ++a) {
                int sd = start_bit(&x, c, a) ? -1 : +1;      /* explicit side */
                int64_t q[3] = {c[0], c[1], c[2]};
                q[a] += sd;
                if (inside(g, q)) e = fma(face_between(g, c, a, sd), xold[lin(g, q)], e);
            }
            alpha[i] = al;
            r0[i] = fma(al, e, (1.0 - w) * xold[i]);
        }
    }
    ctx_free(&x);
    if (st == OR_OK) st = trisolve(g, phase, ov, 0, alpha, r0, xnew, minpiv);
    free(alpha);
    free(r0);
    return st;
}

/* Classical directional SOR written as the textbook in-place
 * loop nest starting at corner `corner_bits`; independent arithmetic order
 * (s = b + sum c u in W,E,S,N,B,F order; u = (1-w) u + (w / a_P) s).  Ignores boxes. */
int or_sor_lex(const or_grid *g, double omega, int corner_bits, double *x, const double *b) {
    int64_t n0 = g->n[0], n1 = g->n[1], n2 = g->n[2];
    for (int64_t kk = 0; kk < n2; ++kk) {
        int64_t k = ((corner_bits >> 2) & 1) ? n2 - 1 - kk : kk;
        for (int64_t jj = 0; jj < n1; ++jj) {
            int64_t j = ((corner_bits >> 1) & 1) ? n1 - 1 - jj : jj;
            for (int64_t ii = 0; ii < n0; ++ii) {
                int64_t i = (corner_bits & 1) ? n0 - 1 - ii : ii;
                int64_t c[3] = {i, j, k};
                double s = b[lin(g, c)];
                for (int a = 0; a < g->dim; ++a)
                    for (int sd = -1; sd <= 1; sd += 2) {
                        int64_t q[3] = {i, j, k};
                        q[a] += sd;
                        if (inside(g, q)) s += face_between(g, c, a, sd) * x[lin(g, q)];
                    }
                int64_t p = lin(g, c);
                x[p] = (1.0 - omega) * x[p] + (omega / a_p(g, c)) * s;
            }
        }
    }
    return OR_OK;
}

/* y = A x  (PAPER eq d2d, 426-428; 1D eq d1d, 184), evaluated as
 *   s = a_P x_p;  s = fma(-c_pq, x_q, s) over neighbours in axis order (-, +)   (R-7) */
void or_apply_A(const or_grid *g, const double *xv, double *y) {
    int64_t N = n_nodes(g);
    for (int64_t i = 0; i < N; ++i) {
        int64_t c[3];
        coords_of(g, i, c);
        double s = a_p(g, c) * xv[i];
        for (int a = 0; a < g->dim; ++a)
            for (int sd = -1; sd <= 1; sd += 2) {
                int64_t q[3] = {c[0], c[1], c[2]};
                q[a] += sd;
                if (inside(g, q)) s = fma(-face_between(g, c, a, sd), xv[lin(g, q)], s);
            }
        y[i] = s;
    }
}

/* Accurate dot product: error-free transformations (TwoProd by fma, TwoSum) accumulate
 * sum a_i b_i in double-double (~106 bits) before the final rounding, so the value is the
 * correctly rounded exact sum except in pathological near-tie cases. */
typedef struct { double hi, lo; } dd_t;

static void dd_add(dd_t *s, double p) {
    double t = s->hi + p;
    double bp = t - s->hi;
    double err = (s->hi - (t - bp)) + (p - bp);
    s->hi = t;
    s->lo += err;
}

static double dot_dd(int64_t N, const double *a, const double *b) {
    dd_t s = {0.0, 0.0};
    for (int64_t i = 0; i < N; ++i) {
        double p = a[i] * b[i];
        double e = fma(a[i], b[i], -p);
        dd_add(&s, p);
        s.lo += e;
    }
    return s.hi + s.lo;
}

/* ||b - A x||_2 / ||b||_2 (stop test of the configs; replaces the paper's L1 error) */
double or_relres(const or_grid *g, const double *xv, const double *b) {
    int64_t N = n_nodes(g);
    double *y = (double *)malloc(sizeof(double) * (size_t)N);
    if (!y) return -1.0;
    or_apply_A(g, xv, y);
    for (int64_t i = 0; i < N; ++i) y[i] = b[i] - y[i];
    double rr = dot_dd(N, y, y), bb = dot_dd(N, b, b);
    free(y);
    return bb > 0.0 ? sqrt(rr) / sqrt(bb) : sqrt(rr);
}

/* ---------------------------------------------------------------- ILU(0)
 * PAPER:911-922 claims one SGS pass on an n-diagonal matrix equals ILU(0) and that the
 * decomposed sweep therefore gives a parallel ILU(0).  Reading R-C (SURVEY §8(c) C-ILU):
 *   D~_p = a_P,p - sum_{q implicit for p, same box} c_pq^2 / D~_q   (wavefront order, phase k0)
 * stored as invD = 1/D~.  Factor in d order; the formula is d = fma(-c*c, invD_q, d). */
int or_ilu0_factor(const or_grid *g, int64_t phase, int ov, double *invD) {
    ctx_t x;
    int st = ctx_init(&x, g, phase, ov);
    int64_t N = n_nodes(g);
    int64_t *order = NULL, *cnt = NULL, *dval = NULL;
    unsigned char *done = NULL;
    if (st != OR_OK) goto out;
    dval = (int64_t *)malloc(sizeof(int64_t) * (size_t)N);
    order = (int64_t *)malloc(sizeof(int64_t) * (size_t)N);
    done = (unsigned char *)calloc((size_t)N, 1);
    if (!dval || !order || !done) { st = OR_ENOMEM; goto out; }
    int64_t dmax = 0;
    for (int64_t i = 0; i < N; ++i) {
        int64_t c[3];
        coords_of(g, i, c);
        dval[i] = wave_d(&x, c);
        if (dval[i] > dmax) dmax = dval[i];
    }
    cnt = (int64_t *)calloc((size_t)(dmax + 2), sizeof(int64_t));
    if (!cnt) { st = OR_ENOMEM; goto out; }
    for (int64_t i = 0; i < N; ++i) cnt[dval[i] + 1]++;
    for (int64_t d = 0; d <= dmax; ++d) cnt[d + 1] += cnt[d];
    for (int64_t i = 0; i < N; ++i) order[cnt[dval[i]]++] = i;
    for (int64_t t = 0; t < N; ++t) {
        int64_t i = order[t];
        int64_t c[3];
        coords_of(g, i, c);
        double dd = a_p(g, c);
        for (int a = 0; a < g->dim; ++a)
            for (int sd = -1; sd <= 1; sd += 2) {
                int64_t q[3] = {c[0], c[1], c[2]};
                q[a] += sd;
                if (!inside(g, q) || !is_implicit(&x, c, a, sd) || !same_box(&x, c, q)) continue;
                int64_t qi = lin(g, q);
                if (!done[qi]) { st = OR_EORDER; goto out; }
                double f = face_between(g, c, a, sd);
                double t2 = f * f;
                dd = fma(-t2, invD[qi], dd);
            }
        if (!(dd > 0.0)) { st = OR_ESINGULAR; goto out; }
        invD[i] = 1.0 / dd;
        done[i] = 1;
    }
out:
    free(dval); free(order); free(done); free(cnt);
    ctx_free(&x);
    return st;
}

/* pairing: 0 = SYMMETRIC  P = (D~+L) D~^-1 (D~+L)^T
 *          1 = PAPER      P = (D~+L) D~^-1 (D~+U),  U = A_E(k0) = A_I(k0+1) */
static int reversed_bits(int dim, int64_t phase, int ov) { return or_base_bits(dim, phase, ov) ^ ((1 << dim) - 1); }

int or_ilu_apply(const or_grid *g, int64_t phase, int ov, const double *invD, int pairing,
                 const double *r, double *z, double *minpiv) {
    int64_t N = n_nodes(g);
    double *r0 = (double *)malloc(sizeof(double) * (size_t)N);
    double *y = (double *)malloc(sizeof(double) * (size_t)N);
    int st = OR_OK;
    if (!r0 || !y) { st = OR_ENOMEM; goto out; }
    for (int64_t i = 0; i < N; ++i) r0[i] = invD[i] * r[i];          /* (D~ + L) y = r, row-normalised */
    st = trisolve(g, phase, ov, 0, invD, r0, y, minpiv);
    if (st != OR_OK) goto out;
    if (pairing == 0)
        st = trisolve(g, phase, ov, 1, invD, y, z, minpiv);           /* (D~ + L^T) z = D~ y */
    else
        st = trisolve(g, 0, reversed_bits(g->dim, phase, ov), 0, invD, y, z, minpiv);  /* (D~ + U) z = D~ y */
out:
    free(r0);
    free(y);
    return st;
}

/* SSOR / SGS preconditioner:
 *   z = w(2-w) (D + w L^T)^-1 D (D + w L)^-1 r        (SYMMETRIC; PAPER pairing uses U for L^T)
 * computed as y = (D/w + L)^-1 r, then (D/w + L^T) z = ((2-w)/w) D y, row-normalised:
 *   y_p = alpha r_p + alpha sum c y,   z_p = (2-w) y_p + alpha sum c z,   alpha = w / a_P. */
int or_ssor_apply(const or_grid *g, double omega, int64_t phase, int ov, int pairing,
                  const double *r, double *z, double *minpiv) {
    int64_t N = n_nodes(g);
    double *al = (double *)malloc(sizeof(double) * (size_t)N);
    double *r0 = (double *)malloc(sizeof(double) * (size_t)N);
    double *y = (double *)malloc(sizeof(double) * (size_t)N);
    int st = OR_OK;
    if (!al || !r0 || !y) { st = OR_ENOMEM; goto out; }
    for (int64_t i = 0; i < N; ++i) {
        int64_t c[3];
        coords_of(g, i, c);
        al[i] = omega / a_p(g, c);
        r0[i] = al[i] * r[i];
    }
    st = trisolve(g, phase, ov, 0, al, r0, y, minpiv);
    if (st != OR_OK) goto out;
    for (int64_t i = 0; i < N; ++i) r0[i] = (2.0 - omega) * y[i];
    if (pairing == 0)
        st = trisolve(g, phase, ov, 1, al, r0, z, minpiv);
    else
        st = trisolve(g, 0, reversed_bits(g->dim, phase, ov), 0, al, r0, z, minpiv);
out:
    free(al);
    free(r0);
    free(y);
    return st;
}

/* ------------------------------------------------------------------- PCG
 * Preconditioned conjugate gradients (north_star; the paper frames SOR/ILU as Krylov
 * preconditioners).  x0 = 0, r0 = b; stop when ||r||/||b|| < rtol on
 * the recursively updated residual.  precond: 0 none, 1 SSOR(omega), 2 D-ILU(0).
 * flexible != 0 uses the Polak-Ribiere beta = z+.(r+ - r)/(r.z) (needed for the
 * nonsymmetric PAPER pairing).  Dot products are accurate (dot_dd); updates are
 * x = fma(alpha, p, x), r = fma(-alpha, q, r), p = fma(beta, p, z). */
static double dot(int64_t N, const double *a, const double *b) { return dot_dd(N, a, b); }

int or_pcg(const or_grid *g, int precond, double omega, int pairing, int flexible, int64_t phase, int ov,
           double rtol, int maxit, const double *b, double *xo, int *iters, double *relres) {
    int64_t N = n_nodes(g);
    double *r = (double *)calloc((size_t)N, sizeof(double));
    double *z = (double *)calloc((size_t)N, sizeof(double));
    double *p = (double *)calloc((size_t)N, sizeof(double));
    double *q = (double *)calloc((size_t)N, sizeof(double));
    double *rold = (double *)calloc((size_t)N, sizeof(double));
    double *invD = (double *)calloc((size_t)N, sizeof(double));
    int st = OR_OK;
    *iters = 0;
    if (!r || !z || !p || !q || !rold || !invD) { st = OR_ENOMEM; goto out; }
    if (precond == 2) {
        st = or_ilu0_factor(g, phase, ov, invD);
        if (st != OR_OK) goto out;
    }
    for (int64_t i = 0; i < N; ++i) { xo[i] = 0.0; r[i] = b[i]; }
    double bnorm = sqrt(dot(N, b, b));
    if (bnorm == 0.0) { *relres = 0.0; goto out; }
#define APPLY_M(src, dst)                                                             \
    do {                                                                              \
        int sm = OR_OK;                                                               \
        if (precond == 0) memcpy(dst, src, sizeof(double) * (size_t)N);               \
        else if (precond == 1) sm = or_ssor_apply(g, omega, phase, ov, pairing, src, dst, NULL); \
        else sm = or_ilu_apply(g, phase, ov, invD, pairing, src, dst, NULL);          \
        if (sm != OR_OK) { st = sm; goto out; }                                       \
    } while (0)
    APPLY_M(r, z);
    memcpy(p, z, sizeof(double) * (size_t)N);
    double rz = dot(N, r, z);
    *relres = 1.0;
    st = OR_ENOCONV;
    for (int it = 1; it <= maxit; ++it) {
        or_apply_A(g, p, q);
        double pq = dot(N, p, q);
        double al = rz / pq;
        if (flexible) memcpy(rold, r, sizeof(double) * (size_t)N);
        for (int64_t i = 0; i < N; ++i) {
            xo[i] = fma(al, p[i], xo[i]);
            r[i] = fma(-al, q[i], r[i]);
        }
        double rr = dot(N, r, r);
        *iters = it;
        *relres = sqrt(rr) / bnorm;
        if (*relres < rtol) { st = OR_OK; break; }
        APPLY_M(r, z);
        double rzn = dot(N, r, z), be;
        if (flexible) {
            for (int64_t i = 0; i < N; ++i) rold[i] = r[i] - rold[i];
            be = dot(N, z, rold) / rz;
        } else {
            be = rzn / rz;
        }
        rz = rzn;
        for (int64_t i = 0; i < N; ++i) p[i] = fma(be, p[i], z[i]);
    }
#undef APPLY_M
out:
    free(r); free(z); free(p); free(q); free(rold); free(invD);
    return st;
}

/* --------------------------------------------------- coefficient assembly
 * Harmonic-mean face coefficients (PAPER:194-197 1D, 443-448 2D), h^2-scaled:
 *   face_a(p, q) = scale_a * ((2 k_p k_q) / (k_p + k_q))     evaluated as (2.0*kp)*kq / (kp+kq)
 * k_ring has n_a + 2 nodes per used axis (boundary ring included, reading R-12), x fastest. */
void or_faces_from_k(int dim, const int64_t n[3], const double *k_ring, const double scale[3], double *face[3]) {
    int64_t m[3] = {1, 1, 1};
    for (int a = 0; a < dim; ++a) m[a] = n[a] + 2;
    for (int a = 0; a < dim; ++a) {
        int64_t f[3] = {n[0], n[1], n[2]};
        f[a] += 1;
        for (int64_t k = 0; k < f[2]; ++k)
            for (int64_t j = 0; j < f[1]; ++j)
                for (int64_t i = 0; i < f[0]; ++i) {
                    /* face between node c - e_a and node c, c = (i,j,k) interior coords; ring idx = c + 1 */
                    int64_t c[3] = {i, j, k};
                    int64_t rq[3], rp[3];
                    for (int t = 0; t < 3; ++t) {
                        rq[t] = (t < dim) ? c[t] + 1 : 0;
                        rp[t] = rq[t];
                    }
                    rp[a] -= 1;
                    double kp = k_ring[rp[0] + m[0] * (rp[1] + m[1] * rp[2])];
                    double kq = k_ring[rq[0] + m[0] * (rq[1] + m[1] * rq[2])];
                    double h = (2.0 * kp) * kq / (kp + kq);
                    face[a][i + f[0] * (j + f[1] * k)] = scale[a] * h;
                }
    }
}

/* diagnostics used by tests: direction bits and wavefront index of every node */
int or_node_info(const or_grid *g, int64_t phase, int ov, int *bits, int64_t *dval) {
    ctx_t x;
    int st = ctx_init(&x, g, phase, ov);
    if (st == OR_OK) {
        int64_t N = n_nodes(g);
        for (int64_t i = 0; i < N; ++i) {
            int64_t c[3];
            coords_of(g, i, c);
            bits[i] = dir_bits(&x, c);
            dval[i] = wave_d(&x, c);
        }
    }
    ctx_free(&x);
    return st;
}

/* diagnostics: histogram of coupled-system (SCC) sizes and of their nonzero counts for the
 * forward sweep at a phase (PAPER:565-567, 682-689 worked 2D example; "32
 * none-zero entries" of the 3D corner system).  hist[s] counts SCCs of size s, nnz[s]
 * sums the nonzeros (diagonal + coupling entries) of those SCC matrices. */
int or_scc_stats(const or_grid *g, int64_t phase, int ov, int64_t hist[9], int64_t nnz[9]) {
    ctx_t x;
    int st = ctx_init(&x, g, phase, ov);
    int64_t N = n_nodes(g);
    unsigned char *seen = (unsigned char *)calloc((size_t)N, 1);
    if (st == OR_OK && !seen) st = OR_ENOMEM;
    for (int s = 0; s < 9; ++s) hist[s] = nnz[s] = 0;
    for (int64_t i = 0; st == OR_OK && i < N; ++i) {
        if (seen[i]) continue;
        int64_t mem[8];
        int k = 1, e = 0;
        mem[0] = i;
        seen[i] = 1;
        for (int h = 0; h < k; ++h) {
            int64_t p[3];
            coords_of(g, mem[h], p);
            for (int a = 0; a < g->dim; ++a)
                for (int sd = -1; sd <= 1; sd += 2) {
                    int64_t q[3] = {p[0], p[1], p[2]};
                    q[a] += sd;
                    if (!inside(g, q)) continue;
                    if (is_implicit(&x, p, a, sd) && is_implicit(&x, q, a, -sd)) {
                        e++;
                        int64_t qi = lin(g, q);
                        if (!seen[qi]) {
                            if (k == 8) { st = OR_EORDER; break; }
                            seen[qi] = 1;
                            mem[k++] = qi;
                        }
                    }
                }
        }
        hist[k]++;
        nnz[k] += k + e;
    }
    free(seen);
    ctx_free(&x);
    return st;
}

/* ------------------------------------------------------- eikonal
 * Parallel fast sweeping for the eikonal equation |grad u| = f on the multi-frontal
 * schedule.  The paper names this application and defers it to a
 * supplementary paper that is not available here, so the local update is the standard
 * fast-sweeping rule (Godunov upwind discretisation, Zhao 2005), reading R-E1 of
 * DESIGN.md:
 *   a = min of the two x-neighbours, b = min of the two y-neighbours (a node outside the
 *   grid counts +inf), fh = f_p * h,
 *   ubar = +inf                                   if min(a, b) = +inf
 *        = min(a, b) + fh                         if |a - b| >= fh
 *        = ((a + b) + sqrt(2 fh^2 - (a - b)^2)) / 2   otherwise,
 *   evaluated as d = a - b, disc = fma(-d, d, 2 (fh fh)), 0.5 ((a + b) + sqrt(disc));
 *   u_p <- min(u_p, ubar).
 * Sources carry u = 0 and keep it (min(0, ubar >= 0) = 0); every other node starts +inf.
 * The decomposed sweep takes neighbours' NEW values on the start side of the node's box
 * and OLD values on the end side (exactly the implicit / explicit split of the SOR sweep,
 * reading R-E2), so the coupled sets at start-start faces are the SOR sweep's SCCs.  A
 * coupled set is solved exactly (reading R-E3) by the ordered (Dijkstra-like) procedure
 * the causality of the Godunov update allows: every unfixed member gets the candidate
 * min(u_old, ubar) with fixed members at their values and unfixed ones at +inf; the member
 * with the smallest candidate (ties: lowest global index) is fixed; repeat.  The smallest
 * member of the exact solution cannot depend on larger members, so this is the exact
 * solution of the set's equations.  1D uses a alone: ubar = a + fh.  2D (and 1D) only. */
static double eik_godunov(int dim, double a, double b, double fh) {
    if (dim == 1) return a + fh;           /* (+inf + fh = +inf) */
    double m = a < b ? a : b;
    if (m == INFINITY) return INFINITY;
    if (fabs(a - b) >= fh) return m + fh;  /* (also when exactly one of a, b is +inf) */
    double d = a - b;
    double disc = fma(-d, d, 2.0 * (fh * fh));
    return 0.5 * ((a + b) + sqrt(disc));
}

/* value of neighbour q of p as the decomposed sweep sees it: +inf outside the grid; inside
 * a set: the fixed value or +inf; otherwise new (implicit for p) or old */
static double eik_nb(const ctx_t *x, const int64_t p[3], int a, int sd, const double *uold, const double *unew,
                     const unsigned char *done, const int64_t *mem, const int *fixed, const double *val, int k,
                     int *err) {
    const or_grid *g = x->g;
    int64_t q[3] = {p[0], p[1], p[2]};
    q[a] += sd;
    if (!inside(g, q)) return INFINITY;
    int64_t qi = lin(g, q);
    for (int m = 0; m < k; ++m)
        if (mem[m] == qi) return fixed[m] ? val[m] : INFINITY;
    if (is_implicit(x, p, a, sd)) {
        if (!done[qi]) *err = OR_EORDER;
        return unew[qi];
    }
    return uold[qi];
}

/* One decomposed eikonal sweep at phase k (2D / 1D): uold -> unew, slowness f > 0, spacing h. */
int or_eik_sweep(const or_grid *g, int64_t phase, int ov, const double *f, double h, const double *uold,
                 double *unew) {
    if (g->dim > 2) return OR_EINVAL;
    ctx_t x;
    int st = ctx_init(&x, g, phase, ov);
    int64_t N = n_nodes(g);
    int64_t *dval = NULL, *order = NULL, *cnt = NULL;
    unsigned char *done = NULL;
    if (st != OR_OK) goto out;
    dval = (int64_t *)malloc(sizeof(int64_t) * (size_t)N);
    order = (int64_t *)malloc(sizeof(int64_t) * (size_t)N);
    done = (unsigned char *)calloc((size_t)N, 1);
    if (!dval || !order || !done) { st = OR_ENOMEM; goto out; }
    int64_t dmax = 0;
    for (int64_t i = 0; i < N; ++i) {
        int64_t c[3];
        coords_of(g, i, c);
        dval[i] = wave_d(&x, c);
        if (dval[i] > dmax) dmax = dval[i];
    }
    cnt = (int64_t *)calloc((size_t)(dmax + 2), sizeof(int64_t));
    if (!cnt) { st = OR_ENOMEM; goto out; }
    for (int64_t i = 0; i < N; ++i) cnt[dval[i] + 1]++;
    for (int64_t d = 0; d <= dmax; ++d) cnt[d + 1] += cnt[d];
    for (int64_t i = 0; i < N; ++i) order[cnt[dval[i]]++] = i;
    for (int64_t t = 0; t < N; ++t) {
        int64_t i = order[t];
        if (done[i]) continue;
        /* the coupled set of i: closure under mutual implicit neighbours (as trisolve) */
        int64_t mem[8];
        int k = 1;
        mem[0] = i;
        for (int hh = 0; hh < k; ++hh) {
            int64_t p[3];
            coords_of(g, mem[hh], p);
            for (int a = 0; a < g->dim; ++a)
                for (int sd = -1; sd <= 1; sd += 2) {
                    int64_t q[3] = {p[0], p[1], p[2]};
                    q[a] += sd;
                    if (!inside(g, q)) continue;
                    if (is_implicit(&x, p, a, sd) && is_implicit(&x, q, a, -sd)) {
                        int64_t qi = lin(g, q);
                        int seen = 0;
                        for (int m = 0; m < k; ++m) seen |= (mem[m] == qi);
                        if (!seen) {
                            if (k == 8) { st = OR_EORDER; goto out; }
                            mem[k++] = qi;
                        }
                    }
                }
        }
        for (int a1 = 1; a1 < k; ++a1)
            for (int b1 = a1; b1 > 0 && mem[b1 - 1] > mem[b1]; --b1) {
                int64_t tmp = mem[b1]; mem[b1] = mem[b1 - 1]; mem[b1 - 1] = tmp;
            }
        int fixed[8] = {0};
        double val[8];
        for (int round = 0; round < k; ++round) {
            int best = -1;
            double cbest = 0.0;
            for (int m = 0; m < k; ++m) {
                if (fixed[m]) continue;
                int64_t p[3];
                coords_of(g, mem[m], p);
                int err = OR_OK;
                double av = INFINITY, bv = INFINITY;
                for (int sd = -1; sd <= 1; sd += 2) {
                    double v = eik_nb(&x, p, 0, sd, uold, unew, done, mem, fixed, val, k, &err);
                    if (v < av) av = v;
                    if (g->dim > 1) {
                        double w = eik_nb(&x, p, 1, sd, uold, unew, done, mem, fixed, val, k, &err);
                        if (w < bv) bv = w;
                    }
                }
                if (err != OR_OK) { st = err; goto out; }
                double ub = eik_godunov(g->dim, av, bv, f[mem[m]] * h);
                double c = uold[mem[m]] < ub ? uold[mem[m]] : ub;
                if (best < 0 || c < cbest) { best = m; cbest = c; }
            }
            fixed[best] = 1;
            val[best] = cbest;
        }
        for (int m = 0; m < k; ++m) {
            unew[mem[m]] = val[m];
            done[mem[m]] = 1;
        }
    }
out:
    free(dval); free(order); free(done); free(cnt);
    ctx_free(&x);
    return st;
}

/* Classical fast sweeping (Zhao 2005): the textbook in-place Gauss-Seidel loop nest from
 * corner `corner_bits` (bit a set = axis a descending), u <- min(u, ubar) with the current
 * values of all neighbours.  Ignores boxes; independent of or_eik_sweep's machinery. */
int or_eik_classical(const or_grid *g, int corner_bits, const double *f, double h, double *u) {
    if (g->dim > 2) return OR_EINVAL;
    int64_t n0 = g->n[0], n1 = g->n[1];
    for (int64_t jj = 0; jj < n1; ++jj) {
        int64_t j = ((corner_bits >> 1) & 1) ? n1 - 1 - jj : jj;
        for (int64_t ii = 0; ii < n0; ++ii) {
            int64_t i = (corner_bits & 1) ? n0 - 1 - ii : ii;
            int64_t p = i + n0 * j;
            double a = INFINITY, b = INFINITY;
            if (i > 0 && u[p - 1] < a) a = u[p - 1];
            if (i < n0 - 1 && u[p + 1] < a) a = u[p + 1];
            if (g->dim > 1) {
                if (j > 0 && u[p - n0] < b) b = u[p - n0];
                if (j < n1 - 1 && u[p + n0] < b) b = u[p + n0];
            }
            double ub = eik_godunov(g->dim, a, b, f[p] * h);
            if (ub < u[p]) u[p] = ub;
        }
    }
    return OR_OK;
}

/* ------------------------------------------------ nine-point molecule
 * "the extension of our algorithm for nine-point or higher order central stencils is
 * straightforward ... the size of local systems to be solved will be also increased"
 * (PAPER:702-707).  2D operator (A u)_p = a_P u_p - sum_{8 neighbours q} c_pq u_q with
 * the axis faces of the grid (face[0], face[1]) and two diagonal coefficient arrays of
 * shape (n0+1) x (n1+1):
 *   dd[c] couples (c_x-1, c_y-1) and c       (SW-NE diagonal of the cell with corner c)
 *   da[c] couples (c_x-1, c_y) and (c_x, c_y-1)   (SE-NW diagonal)
 * a_P = ((F_W + F_E) + (F_S + F_N)) + ((D_SW + D_NE) + (D_SE + D_NW)) + beta.
 * Reading R-N3: the paper's classification, extended to diagonal neighbours --
 * q is IMPLICIT (new value) for p iff q lies on the start side of p's box along every axis
 * in which they differ, else explicit (old value).  For the five-point stencil this is the
 * SOR sweep above; for nine points a box takes W, S, SW new and E, N, NE, SE, NW old (the
 * frontal order: SE and NW sit on p's own front), and at a start corner the four boxes'
 * corner nodes become mutually implicit along the diagonals too: the corner set grows from
 * the 4-cycle to a dense 4 x 4 (the "increased local systems").  Neighbour order of every
 * sum: W, E, S, N, SW, SE, NW, NE; per-node formula and coupled-set elimination as R-7/R-8. */
static const int NB9[8][2] = {{-1, 0}, {1, 0}, {0, -1}, {0, 1}, {-1, -1}, {1, -1}, {-1, 1}, {1, 1}};

static double coef9(const or_grid *g, const double *dd, const double *da, const int64_t c[3], int k) {
    int dx = NB9[k][0], dy = NB9[k][1];
    if (dy == 0) return face_between(g, c, 0, dx);
    if (dx == 0) return face_between(g, c, 1, dy);
    int64_t m0 = g->n[0] + 1;
    if (dx == dy) {                               /* SW (-1,-1) or NE (+1,+1): dd at the upper corner */
        int64_t cx = c[0] + (dx > 0), cy = c[1] + (dy > 0);
        return dd[cx + m0 * cy];
    }
    /* SE (+1,-1): da[(x+1, y)];  NW (-1,+1): da[(x, y+1)] */
    int64_t cx = c[0] + (dx > 0), cy = c[1] + (dy > 0);
    return da[cx + m0 * cy];
}

static double a_p9(const or_grid *g, const double *dd, const double *da, const int64_t c[3]) {
    double s = (coef9(g, dd, da, c, 0) + coef9(g, dd, da, c, 1)) + (coef9(g, dd, da, c, 2) + coef9(g, dd, da, c, 3));
    double t = (coef9(g, dd, da, c, 4) + coef9(g, dd, da, c, 7)) + (coef9(g, dd, da, c, 5) + coef9(g, dd, da, c, 6));
    return (s + t) + g->beta;
}

static int implicit9(const ctx_t *x, const int64_t p[3], int k) {
    int dx = NB9[k][0], dy = NB9[k][1];
    return (dx == 0 || is_implicit(x, p, 0, dx)) && (dy == 0 || is_implicit(x, p, 1, dy));
}

/* One decomposed nine-point SOR sweep at phase k (2D). */
int or_sweep9(const or_grid *g, const double *dd, const double *da, const double *omega, int n_omega, int64_t phase,
              int ov, const double *xold, const double *b, double *xnew, double *minpiv) {
    if (g->dim != 2) return OR_EINVAL;
    ctx_t x;
    int st = ctx_init(&x, g, phase, ov);
    int64_t N = n_nodes(g);
    double *alpha = (double *)malloc(sizeof(double) * (size_t)N);
    double *r0 = (double *)malloc(sizeof(double) * (size_t)N);
    int64_t *dval = (int64_t *)malloc(sizeof(int64_t) * (size_t)N);
    int64_t *order = (int64_t *)malloc(sizeof(int64_t) * (size_t)N);
    unsigned char *done = (unsigned char *)calloc((size_t)N, 1);
    int64_t *cnt = NULL;
    if (st != OR_OK) goto out;
    if (!alpha || !r0 || !dval || !order || !done) { st = OR_ENOMEM; goto out; }
    /* explicit parts: r0 = fma(alpha, b + sum_explicit c u_old, (1 - w) u_old) */
    for (int64_t i = 0; i < N; ++i) {
        int64_t c[3];
        coords_of(g, i, c);
        double w = omega[n_omega == 1 ? 0 : dir_bits(&x, c)];
        double al = w / a_p9(g, dd, da, c);
        double e = b[i];
        for (int k = 0; k < 8; ++k) {
            int64_t q[3] = {c[0] + NB9[k][0], c[1] + NB9[k][1], c[2]};
            if (!inside(g, q) || implicit9(&x, c, k)) continue;
            e = fma(coef9(g, dd, da, c, k), xold[lin(g, q)], e);
        }
        alpha[i] = al;
        r0[i] = fma(al, e, (1.0 - w) * xold[i]);
    }
    /* fronts: implicit neighbours lie on earlier fronts or in the node's coupled set */
    int64_t dmax = 0;
    for (int64_t i = 0; i < N; ++i) {
        int64_t c[3];
        coords_of(g, i, c);
        dval[i] = wave_d(&x, c);
        if (dval[i] > dmax) dmax = dval[i];
    }
    cnt = (int64_t *)calloc((size_t)(dmax + 2), sizeof(int64_t));
    if (!cnt) { st = OR_ENOMEM; goto out; }
    for (int64_t i = 0; i < N; ++i) cnt[dval[i] + 1]++;
    for (int64_t d = 0; d <= dmax; ++d) cnt[d + 1] += cnt[d];
    for (int64_t i = 0; i < N; ++i) order[cnt[dval[i]]++] = i;
    for (int64_t t = 0; t < N; ++t) {
        int64_t i = order[t];
        if (done[i]) continue;
        int64_t mem[8];
        int k = 1;
        mem[0] = i;
        for (int h = 0; h < k; ++h) {              /* closure under mutual implicit neighbours */
            int64_t p[3];
            coords_of(g, mem[h], p);
            for (int kk = 0; kk < 8; ++kk) {
                int64_t q[3] = {p[0] + NB9[kk][0], p[1] + NB9[kk][1], p[2]};
                if (!inside(g, q) || !implicit9(&x, p, kk)) continue;
                int back = -1;
                for (int k2 = 0; k2 < 8; ++k2)
                    if (NB9[k2][0] == -NB9[kk][0] && NB9[k2][1] == -NB9[kk][1]) back = k2;
                if (!implicit9(&x, q, back)) continue;
                int64_t qi = lin(g, q);
                int seen = 0;
                for (int m = 0; m < k; ++m) seen |= (mem[m] == qi);
                if (!seen) {
                    if (k == 8) { st = OR_EORDER; goto out; }
                    mem[k++] = qi;
                }
            }
        }
        for (int a1 = 1; a1 < k; ++a1)
            for (int b1 = a1; b1 > 0 && mem[b1 - 1] > mem[b1]; --b1) {
                int64_t tmp = mem[b1]; mem[b1] = mem[b1 - 1]; mem[b1 - 1] = tmp;
            }
        double M[8][8], rhs[8], u[8];
        for (int p = 0; p < k; ++p) {
            int64_t pc[3];
            coords_of(g, mem[p], pc);
            for (int q = 0; q < k; ++q) M[p][q] = (p == q) ? 1.0 : 0.0;
            double acc = r0[mem[p]];
            for (int kk = 0; kk < 8; ++kk) {
                int64_t qc[3] = {pc[0] + NB9[kk][0], pc[1] + NB9[kk][1], pc[2]};
                if (!inside(g, qc) || !implicit9(&x, pc, kk)) continue;
                int64_t qi = lin(g, qc);
                double m = alpha[mem[p]] * coef9(g, dd, da, pc, kk);
                int inscc = -1;
                for (int q = 0; q < k; ++q)
                    if (mem[q] == qi) inscc = q;
                if (inscc >= 0) {
                    M[p][inscc] = -m;
                } else {
                    if (!done[qi]) { st = OR_EORDER; goto out; }
                    acc = fma(m, xnew[qi], acc);
                }
            }
            rhs[p] = acc;
        }
        if (k == 1) {
            u[0] = rhs[0];
        } else {
            st = ge_solve(k, M, rhs, u, minpiv);
            if (st != OR_OK) goto out;
        }
        for (int p = 0; p < k; ++p) {
            xnew[mem[p]] = u[p];
            done[mem[p]] = 1;
        }
    }
out:
    free(alpha); free(r0); free(dval); free(order); free(done); free(cnt);
    ctx_free(&x);
    return st;
}

/* Textbook frontal nine-point SOR from corner `corner_bits`, one box: fronts d = distance from
 * the corner in order; every node of front d from W, S, SW of the new iterate (earlier fronts)
 * and E, N, NE, SE, NW of the old one (its own and later fronts):
 *   u_p = (1 - w) u_p + (w / a_P) (b_p + sum_q c_pq u_q)      (plain sums, no fma).
 * Independent of or_sweep9's machinery; ignores boxes. */
int or_sor9_frontal(const or_grid *g, const double *dd, const double *da, double omega, int corner_bits,
                    const double *xold, const double *b, double *xnew) {
    if (g->dim != 2) return OR_EINVAL;
    int64_t n0 = g->n[0], n1 = g->n[1];
    int sx = corner_bits & 1, sy = (corner_bits >> 1) & 1;
    for (int64_t d = 0; d <= (n0 - 1) + (n1 - 1); ++d)
        for (int64_t jj = 0; jj < n1; ++jj) {
            int64_t ii = d - jj;
            if (ii < 0 || ii >= n0) continue;
            int64_t i = sx ? n0 - 1 - ii : ii, j = sy ? n1 - 1 - jj : jj;
            int64_t c[3] = {i, j, 0};
            double s = b[lin(g, c)];
            for (int k = 0; k < 8; ++k) {
                int dx = NB9[k][0], dy = NB9[k][1];
                int64_t q[3] = {i + dx, j + dy, 0};
                if (!inside(g, q)) continue;
                /* in sweep coordinates: the neighbour is new iff it lies back along every differing axis */
                int ldx = sx ? -dx : dx, ldy = sy ? -dy : dy;
                int isnew = (ldx <= 0 && ldy <= 0);
                s += coef9(g, dd, da, c, k) * (isnew ? xnew[lin(g, q)] : xold[lin(g, q)]);
            }
            int64_t p = lin(g, c);
            xnew[p] = (1.0 - omega) * xold[p] + (omega / a_p9(g, dd, da, c)) * s;
        }
    return OR_OK;
}
