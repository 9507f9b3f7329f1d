// tri3t.cuh -- second phase of the transposed (SYMMETRIC-pairing) triangular solve in 3D, sm_100a
// (DESIGN R-C; SURVEY §8(a) a11-a12, §8(c) C-ILU).
//
// The backward factor of the SYMMETRIC pairing solves (D/alpha + A_I^T) z = r0:
//     z_p = coef src_p + sum_{q : p implicit for q} alpha_p c_pq z_q .
// Phase 1 (k_sweep3 run from the far corner with the coupling off) is exact for every node outside
// a coupled set.  The coupled sets are recomputed here by degree, one launch each, because a set
// of degree j reads sets of degree j - 1 that neighbouring boxes compute:
//   NA = 1: the pairs of the three start-face sheets, a reverse 2D wavefront per sheet;
//   NA = 2: the three edge chains of 4-sets, reversed;
//   NA = 3: the corner set.
// One warp per box, one lane per sheet line / edge.  The member rows are built in the order of
// the oracle's transposed solve (axes ascending, global -1 side before +1; the partner across a
// coupled face goes into the matrix) and eliminated without pivoting in ascending global index
// (DESIGN R-8), so the results are bitwise those of the oracle (and of k_generic's M_T2 pass).
#pragma once
#include "common.cuh"

namespace sw {

struct Tri3tArgs {
    Geo G;
    int base;                   // direction bits of the forward pass (phase k0)
    double omega;               // SSOR: alpha = omega / a_P
    double coef;                // r0 = coef src
    const double *invd;         // ILU: alpha = 1/D~ (null for SSOR)
    const double *src;          // phase-1 right-hand side (y)
    const double *f0, *f1, *f2; // faces (null: Poisson)
    double *z;                  // phase-1 result, coupled sets corrected in place
    int *flag;
};

// box parity bit of global coordinate c along axis a (global coordinates fit in 32 bits)
// (a float reciprocal instead of an integer division: the quotient (c + 1/2) / T is exact to the
// integer part for c < 2^22)
__device__ __forceinline__ int box_bit(const Tri3tArgs &A, int a, int64_t c) {
    return __float2int_rz(((float)c + 0.5f) * __frcp_rn((float)A.G.T[a])) & 1;
}

template <int NA>
__device__ __forceinline__ void tri3t_solve(const Tri3tArgs &A, const int64_t gl[3], int mask) {
    const Geo &G = A.G;
    constexpr int k = 1 << NA;
    int bitof[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) bitof[a] = __popc(mask & ((1 << a) - 1));
    const int64_t S[3] = {1, G.P0, G.P01};
    const double *const F[3] = {A.f0, A.f1, A.f2};
    double M[k][k], rhs[k], u[k];
    int64_t ix[k];
#pragma unroll
    for (int p = 0; p < k; ++p) {
        int64_t g[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) g[a] = gl[a] + (((mask >> a) & 1) ? ((p >> bitof[a]) & 1) : 0);
        const int64_t i = gidx(G, g[0], g[1], g[2]);
        ix[p] = i;
        // faces toward -a and +a of this member
        double fm[3], fp[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            fm[a] = G.poisson ? 1.0 : F[a][i];
            fp[a] = G.poisson ? 1.0 : F[a][i + S[a]];
        }
        double al;
        if (A.invd) {
            al = A.invd[i];
        } else {
            const double ap = (((fm[0] + fp[0]) + (fm[1] + fp[1])) + (fm[2] + fp[2])) + G.beta;
            al = div_rn(A.omega, ap);               // = A.omega / ap (IEEE), no slow-path branch
        }
        double acc = A.coef * A.src[i];
#pragma unroll
        for (int q = 0; q < k; ++q) M[p][q] = (p == q) ? 1.0 : 0.0;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
#pragma unroll
            for (int sd = -1; sd <= 1; sd += 2) {
                const int64_t qa = g[a] + sd;
                if (qa < 0 || qa >= G.ng[a]) continue;              // outside the domain
                // p is implicit for q = p + sd e_a iff q's box starts at the side facing p
                const int sq = ((A.base >> a) & 1) ^ box_bit(A, a, qa);
                if (sq != (sd < 0 ? 1 : 0)) continue;
                const double m = al * (sd < 0 ? fm[a] : fp[a]);
                int in = -1;
                if ((mask >> a) & 1) {
                    const int bit = bitof[a];
                    const int64_t other = gl[a] + (((p >> bit) & 1) ^ 1);   // the partner's coordinate
                    if (other == qa) in = p ^ (1 << bit);
                }
                if (in >= 0) {
#pragma unroll
                    for (int c = 0; c < k; ++c)
                        if (c == in) M[p][c] = -m;
                } else {
                    acc = fma(m, A.z[i + sd * S[a]], acc);
                }
            }
        }
        rhs[p] = acc;
    }
    double inv[k];
#pragma unroll
    for (int p = 0; p < k; ++p) {
        const double piv = M[p][p];
        if (!(fabs(piv) >= 1e-14)) atomicOr(A.flag, 1);
        inv[p] = div_rn(1.0, piv);
#pragma unroll
        for (int q = p + 1; q < k; ++q) {
            const double l = M[q][p] * inv[p];
#pragma unroll
            for (int j = p + 1; j < k; ++j) M[q][j] = fma(-l, M[p][j], M[q][j]);
            rhs[q] = fma(-l, rhs[p], rhs[q]);
        }
    }
#pragma unroll
    for (int p = k - 1; p >= 0; --p) {
        double s = rhs[p];
#pragma unroll
        for (int j = p + 1; j < k; ++j) s = fma(-M[p][j], u[j], s);
        u[p] = s * inv[p];
    }
#pragma unroll
    for (int p = 0; p < k; ++p) A.z[ix[p]] = u[p];
}

// Row of member p alone (the same operations as tri3t_solve's member loop): rhs and the matrix row.
template <int NA>
__device__ __forceinline__ void tri3t_row(const Tri3tArgs &A, const int64_t gl[3], int mask, int p, double &rhs,
                                          double (&Mr)[1 << NA], int64_t &ix) {
    const Geo &G = A.G;
    constexpr int k = 1 << NA;
    int bitof[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) bitof[a] = __popc(mask & ((1 << a) - 1));
    const int64_t S[3] = {1, G.P0, G.P01};
    const double *const F[3] = {A.f0, A.f1, A.f2};
    int64_t g[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) g[a] = gl[a] + (((mask >> a) & 1) ? ((p >> bitof[a]) & 1) : 0);
    const int64_t i = gidx(G, g[0], g[1], g[2]);
    ix = i;
    double fm[3], fp[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        fm[a] = G.poisson ? 1.0 : F[a][i];
        fp[a] = G.poisson ? 1.0 : F[a][i + S[a]];
    }
    double al;
    if (A.invd) {
        al = A.invd[i];
    } else {
        const double ap = (((fm[0] + fp[0]) + (fm[1] + fp[1])) + (fm[2] + fp[2])) + G.beta;
        al = div_rn(A.omega, ap);               // = A.omega / ap (IEEE), no slow-path branch
    }
    double acc = A.coef * A.src[i];
#pragma unroll
    for (int q = 0; q < k; ++q) Mr[q] = (p == q) ? 1.0 : 0.0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
#pragma unroll
        for (int sd = -1; sd <= 1; sd += 2) {
            const int64_t qa = g[a] + sd;
            if (qa < 0 || qa >= G.ng[a]) continue;
            const int sq = ((A.base >> a) & 1) ^ box_bit(A, a, qa);
            if (sq != (sd < 0 ? 1 : 0)) continue;
            const double m = al * (sd < 0 ? fm[a] : fp[a]);
            int in = -1;
            if ((mask >> a) & 1) {
                const int bit = bitof[a];
                const int64_t other = gl[a] + (((p >> bit) & 1) ^ 1);
                if (other == qa) in = p ^ (1 << bit);
            }
            if (in >= 0) {
#pragma unroll
                for (int c = 0; c < k; ++c)
                    if (c == in) Mr[c] = -m;
            } else {
                acc = fma(m, A.z[i + sd * S[a]], acc);
            }
        }
    }
    rhs = acc;
}

// Gaussian elimination of a gathered k x k set (rows in rank order) as in tri3t_solve.
template <int K>
__device__ __forceinline__ void tri3t_ge(double (&M)[K][K], double (&rhs)[K], double (&u)[K], int *flag, bool report) {
    double inv[K];
#pragma unroll
    for (int p = 0; p < K; ++p) {
        const double piv = M[p][p];
        if (report && !(fabs(piv) >= 1e-14)) atomicOr(flag, 1);
        inv[p] = div_rn(1.0, piv);
#pragma unroll
        for (int q = p + 1; q < K; ++q) {
            const double l = M[q][p] * inv[p];
#pragma unroll
            for (int j = p + 1; j < K; ++j) M[q][j] = fma(-l, M[p][j], M[q][j]);
            rhs[q] = fma(-l, rhs[p], rhs[q]);
        }
    }
#pragma unroll
    for (int p = K - 1; p >= 0; --p) {
        double s = rhs[p];
#pragma unroll
        for (int j = p + 1; j < K; ++j) s = fma(-M[p][j], u[j], s);
        u[p] = s * inv[p];
    }
}

template <int NA>
__global__ void __launch_bounds__(32) k_tri3t(Tri3tArgs A) {
    SW_JITTER_POINT();
    const Geo &G = A.G;
    const int64_t t = blockIdx.x;
    int64_t R[3] = {t % G.nt[0], (t / G.nt[0]) % G.nt[1], t / ((int64_t)G.nt[0] * G.nt[1])};
    int s[3], cpl[3];
    int64_t lo_g[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        R[a] += G.toff[a];
        s[a] = ((A.base >> a) & 1) ^ (int)(R[a] & 1);
        cpl[a] = s[a] ? (R[a] < G.ntg[a] - 1) : (R[a] > 0);
        lo_g[a] = R[a] * G.T[a];
    }
    const int T0 = G.T[0], T1 = G.T[1], T2 = G.T[2];
    const int tmax = T0 > T1 ? (T0 > T2 ? T0 : T2) : (T1 > T2 ? T1 : T2);
    // Every set is shared by the 2 / 4 / 8 boxes whose start corners meet at it, and each of them
    // would compute it (bitwise the same values: the rows use global indices only).  On one rank
    // only the box with the lowest index along every set axis does (it starts at the high end of
    // each: s = 1); over slabs every box still computes its sets, because a set across the slab
    // boundary must be written on both ranks.
    const bool single = G.nt[2] == G.ntg[2];
    int own[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) own[a] = cpl[a] && (!single || s[a] == 1);
    if (NA == 3) {                                   // the corner set: one lane
        if (threadIdx.x == 0 && own[0] && own[1] && own[2]) {
            int64_t gl[3];
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                const int64_t g = s[a] ? (lo_g[a] + G.T[a] - 1) : lo_g[a];
                const int64_t other = s[a] ? (lo_g[a] + G.T[a]) : (lo_g[a] - 1);
                gl[a] = other < g ? other : g;
            }
            tri3t_solve<3>(A, gl, 7);
        }
        return;
    }
    // NA = 1: lane pairs (2 members) per sheet line; NA = 2: lane quads (4 members) per edge.  Every
    // lane builds its member's row, the group gathers the rows by shuffles and eliminates them
    // redundantly, and each lane writes its member.
    constexpr int K = 1 << NA;
    const int p = threadIdx.x & (K - 1);
    const int grp = threadIdx.x / K;                    // 16 sheet lines / 8 edge groups per pass
    const int n0 = own[0] ? T2 : 0, n1 = own[1] ? T2 : 0, n2 = own[2] ? T1 : 0;
    const int nlines = NA == 1 ? n0 + n1 + n2 : 3;
    const int dmax = NA == 2 ? tmax - 1 : T0 - 1 + (T1 > T2 ? T1 : T2) - 1;
    // geometry of line `ln` at step d: active?, rank-0 corner gl of the set, set axes, and the
    // line's walk / fixed axes
    auto geom = [&](int d, int ln, bool &ok, int64_t (&gl)[3], int &mask, int &walk, int &fixax) {
        int fa = -1, fixv = 0;
        walk = 0;
        fixax = 0;
        if (NA == 1) {
            if (ln < n0) { fa = 0; fixax = 2; fixv = ln; walk = 1; }
            else if ((ln -= n0) < n1) { fa = 1; fixax = 2; fixv = ln; walk = 0; }
            else if ((ln -= n1) < n2) { fa = 2; fixax = 1; fixv = ln; walk = 0; }
        } else {
            if (ln < 3 && own[(ln + 1) % 3] && own[(ln + 2) % 3]) { fa = ln; walk = ln; fixax = -1; }
        }
        ok = fa >= 0;
        int l[3] = {0, 0, 0};
        if (ok && NA == 1) {
            l[fixax] = fixv;
            l[walk] = d - fixv;
#pragma unroll
            for (int a = 0; a < 3; ++a)
                if (a != fa && (l[a] < (cpl[a] ? 1 : 0) || l[a] >= G.T[a])) ok = false;
        } else if (ok) {
            l[walk] = d;
            if (d < (cpl[walk] ? 1 : 0) || d >= G.T[walk]) ok = false;
        }
        mask = 0;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            gl[a] = 0;
            if (ok) {
                const int64_t g = s[a] ? (lo_g[a] + G.T[a] - 1 - l[a]) : (lo_g[a] + l[a]);
                gl[a] = g;
                if (cpl[a] && l[a] == 0) {
                    mask |= 1 << a;
                    const int64_t other = s[a] ? (lo_g[a] + G.T[a]) : (lo_g[a] - 1);
                    if (other < gl[a]) gl[a] = other;
                }
            }
        }
    };
    if (nlines <= 32 / K) {
        // Fast path (every line in one pass; 32 x 8 x 4 boxes).  Along a line every member row has
        // the same shape: the partner across each set axis (the matrix entry), the node beyond it
        // (a value of phase 1 or of the previous launch), the next node along the line (this lane's
        // result of the previous step) and, for sheets, the same node of the next line (the result
        // of lane + K in the previous step).  So the row is built from per-line constants and
        // values already in registers, with exactly the operations and order of tri3t_row (axes
        // ascending, one term per axis), and the loads of step d - 1 are issued during step d.
        const int ln = grp;
        bool act;
        int64_t gl0[3];
        int mask, walk, fixax;
        // geometry at the line's first active step (any active d gives the same mask and the
        // same coordinates off the walk axis)
        int fixv = 0, lo_w = 0;
        {
            int l_ln = ln, fa = -1;
            if (NA == 1) {
                if (l_ln < n0) { fa = 0; fixv = l_ln; }
                else if ((l_ln -= n0) < n1) { fa = 1; fixv = l_ln; }
                else if ((l_ln -= n1) < n2) { fa = 2; fixv = l_ln; }
            } else if (ln < 3 && own[(ln + 1) % 3] && own[(ln + 2) % 3]) {
                fa = ln;
            }
            act = fa >= 0;
            int w_ = 0, f_ = 0;
            if (act) {
                if (NA == 1) { w_ = fa == 0 ? 1 : 0; f_ = fa == 2 ? 1 : 2; }
                else w_ = fa;
            }
            lo_w = cpl[w_] ? 1 : 0;
            if (NA == 1 && act && (fixv < (cpl[f_] ? 1 : 0) || fixv >= G.T[f_])) act = false;
            bool okg = false;
            int wk, fx;
            geom(NA == 1 ? lo_w + fixv : lo_w, ln, okg, gl0, mask, wk, fx);
            act = act && okg;
            walk = w_;
            fixax = f_;
        }
        const int Tw = G.T[walk];
        // member coordinates at l[walk] = lo_w, and the per-axis roles
        int bitof[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) bitof[a] = __popc(mask & ((1 << a) - 1));
        int64_t g[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) g[a] = gl0[a] + (((mask >> a) & 1) ? ((p >> bitof[a]) & 1) : 0);
        const int64_t S[3] = {1, G.P0, G.P01};
        const int lw = s[walk] ? -1 : 1;                       // global step of local +1 along the walk
        const int lf = NA == 1 ? (s[fixax] ? -1 : 1) : 0;
        const int64_t istep = lw * S[walk];
        const int64_t i_lo = act ? gidx(G, g[0], g[1], g[2]) : 0;   // member index at l[walk] = lo_w
        const bool fix_term = NA == 1 && act && fixv + 1 < G.T[fixax];
        // set axes: direction of the partner / of the node beyond; the node beyond exists unless
        // the box is one node thick there
        int sdp[3], sdb[3];
        bool bey[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const int b = ((mask >> a) & 1) ? ((p >> bitof[a]) & 1) : 0;
            sdp[a] = b ? -1 : 1;
            sdb[a] = -sdp[a];
            bey[a] = G.T[a] >= 2;
        }
        const double *const F[3] = {A.f0, A.f1, A.f2};
        struct Pre { double src, invd, fm[3], fp[3], zb[3]; };
        auto pref = [&](int64_t i, Pre &P) {
            P.src = A.src[i];
            P.invd = A.invd ? A.invd[i] : 0.0;
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                P.fm[a] = G.poisson ? 1.0 : F[a][i];
                P.fp[a] = G.poisson ? 1.0 : F[a][i + S[a]];
                P.zb[a] = ((mask >> a) & 1) ? A.z[i + sdb[a] * S[a]] : 0.0;
            }
        };
        auto lw_at = [&](int d) { return NA == 1 ? d - fixv : d; };   // l[walk] at step d
        Pre cur, nxt;
        {
            const int l = lw_at(dmax);
            if (act && l >= lo_w && l < Tw) pref(i_lo + (l - lo_w) * istep, cur);
        }
        double prev = 0.0;
        for (int d = dmax; d >= 0; --d) {
            const int l = lw_at(d);
            const bool okc = act && l >= lo_w && l < Tw;
            const int ln1 = l - 1;
            if (d > 0 && act && ln1 >= lo_w && ln1 < Tw) pref(i_lo + (ln1 - lo_w) * istep, nxt);
            const double adj = __shfl_sync(0xffffffffu, prev, (threadIdx.x + K) & 31);   // next line, same member
            double rhs = 0.0, off[NA];
#pragma unroll
            for (int t = 0; t < NA; ++t) off[t] = 0.0;
            if (okc) {
                double al;
                if (A.invd) {
                    al = cur.invd;
                } else {
                    const double ap = (((cur.fm[0] + cur.fp[0]) + (cur.fm[1] + cur.fp[1])) + (cur.fm[2] + cur.fp[2])) + G.beta;
                    al = div_rn(A.omega, ap);               // = A.omega / ap (IEEE), no slow-path branch
                }
                double acc = A.coef * cur.src;
                int t = 0;
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    if ((mask >> a) & 1) {                       // set axis: partner entry, node beyond
                        const double mp = al * (sdp[a] < 0 ? cur.fm[a] : cur.fp[a]);
                        const double mb = al * (sdb[a] < 0 ? cur.fm[a] : cur.fp[a]);
                        // the original loop visits sd = -1 first: the partner entry does not touch acc
                        if (bey[a]) acc = fma(mb, cur.zb[a], acc);
#pragma unroll
                        for (int u = 0; u < NA; ++u)
                            if (u == t) off[u] = -mp;
                        ++t;
                    } else if (a == walk) {
                        if (l + 1 < Tw) acc = fma(al * (lw < 0 ? cur.fm[a] : cur.fp[a]), prev, acc);
                    } else if (fix_term) {                       // NA = 1: the fixed axis
                        acc = fma(al * (lf < 0 ? cur.fm[a] : cur.fp[a]), adj, acc);
                    }
                }
                rhs = acc;
            }
            double Mall[K][K], rall[K], u[K];
            const int src0 = threadIdx.x & ~(K - 1);
#pragma unroll
            for (int q = 0; q < K; ++q) {
                rall[q] = __shfl_sync(0xffffffffu, rhs, src0 + q);
#pragma unroll
                for (int c = 0; c < K; ++c) Mall[q][c] = (c == q) ? 1.0 : 0.0;
#pragma unroll
                for (int tt = 0; tt < NA; ++tt) Mall[q][q ^ (1 << tt)] = __shfl_sync(0xffffffffu, off[tt], src0 + q);
            }
            if (okc) {
                tri3t_ge<K>(Mall, rall, u, A.flag, p == 0);
                double mine = u[0];
#pragma unroll
                for (int c = 1; c < K; ++c)
                    if (c == p) mine = u[c];
                A.z[i_lo + (l - lo_w) * istep] = mine;
                prev = mine;
            }
            cur = nxt;
        }
        return;
    }
    for (int d = dmax; d >= 0; --d) {
        for (int base_ln = 0; base_ln < nlines; base_ln += 32 / K) {
            int ln = base_ln + grp;
            int fa = -1, fixv = 0, walk = 0, fixax = 0;
            if (NA == 1) {
                if (ln < n0) { fa = 0; fixax = 2; fixv = ln; walk = 1; }
                else if ((ln -= n0) < n1) { fa = 1; fixax = 2; fixv = ln; walk = 0; }
                else if ((ln -= n1) < n2) { fa = 2; fixax = 1; fixv = ln; walk = 0; }
            } else {
                if (ln < 3 && own[(ln + 1) % 3] && own[(ln + 2) % 3]) { fa = ln; walk = ln; }
            }
            bool ok = fa >= 0;
            int l[3] = {0, 0, 0};
            if (ok && NA == 1) {
                l[fixax] = fixv;
                l[walk] = d - fixv;
                // the other two coordinates off the coupled start faces (else a set of higher
                // degree) and inside the box
#pragma unroll
                for (int a = 0; a < 3; ++a)
                    if (a != fa && (l[a] < (cpl[a] ? 1 : 0) || l[a] >= G.T[a])) ok = false;
            } else if (ok) {
                l[walk] = d;
                if (d < (cpl[walk] ? 1 : 0) || d >= G.T[walk]) ok = false;
            }
            int64_t gl[3] = {0, 0, 0};
            int mask = 0;
            if (ok) {
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    const int64_t g = s[a] ? (lo_g[a] + G.T[a] - 1 - l[a]) : (lo_g[a] + l[a]);
                    gl[a] = g;
                    if (cpl[a] && l[a] == 0) {
                        mask |= 1 << a;
                        const int64_t other = s[a] ? (lo_g[a] + G.T[a]) : (lo_g[a] - 1);
                        if (other < gl[a]) gl[a] = other;
                    }
                }
            }
            double rhs = 0.0, Mr[K];
            int64_t ix = 0;
#pragma unroll
            for (int c = 0; c < K; ++c) Mr[c] = (c == p) ? 1.0 : 0.0;
            if (ok) tri3t_row<NA>(A, gl, mask, p, rhs, Mr, ix);
            double Mall[K][K], rall[K], u[K];
            const int src0 = threadIdx.x & ~(K - 1);
            // gather the rows: the right-hand side and the NA off-diagonal entries (to the partner
            // across each set axis, p ^ (1 << t)); the rest of every row is the identity's
            double off[NA];
#pragma unroll
            for (int t = 0; t < NA; ++t) {
                off[t] = Mr[0];
#pragma unroll
                for (int c = 1; c < K; ++c)
                    if (c == (p ^ (1 << t))) off[t] = Mr[c];
            }
#pragma unroll
            for (int q = 0; q < K; ++q) {
                rall[q] = __shfl_sync(0xffffffffu, rhs, src0 + q);
#pragma unroll
                for (int c = 0; c < K; ++c) Mall[q][c] = (c == q) ? 1.0 : 0.0;
#pragma unroll
                for (int t = 0; t < NA; ++t) Mall[q][q ^ (1 << t)] = __shfl_sync(0xffffffffu, off[t], src0 + q);
            }
            if (ok) {
                tri3t_ge<K>(Mall, rall, u, A.flag, p == 0);
                double mine = u[0];
#pragma unroll
                for (int c = 1; c < K; ++c)
                    if (c == p) mine = u[c];
                A.z[ix] = mine;
            }
        }
        __syncwarp();
    }
}

inline cudaError_t launch_tri3t(const Tri3tArgs &A, int degree, cudaStream_t s) {
    const unsigned tiles = (unsigned)((int64_t)A.G.nt[0] * A.G.nt[1] * A.G.nt[2]);
    switch (degree) {
        case 1: k_tri3t<1><<<tiles, 32, 0, s>>>(A); break;
        case 2: k_tri3t<2><<<tiles, 32, 0, s>>>(A); break;
        default: k_tri3t<3><<<tiles, 32, 0, s>>>(A); break;
    }
    return cudaGetLastError();
}

}  // namespace sw
