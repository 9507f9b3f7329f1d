// generic.cuh -- level-synchronous tile kernel for every dimension and every mode of
// the decomposed sweep family (SOR sweep, ILU/SSOR forward, PAPER-pairing backward,
// SYMMETRIC-pairing transposed backward in phases, ILU(0) factor).
//
// One CTA = one box (tile).  The box's work is processed wavefront by wavefront
// (d = sum of distances to the box's start corner, "frontal" order,
// 524-680), one __syncthreads per wavefront.  Coupled systems (PAPER:289-304, 578-680,
// 884-895) appear as sets of 2^j nodes straddling the j start faces through the box's
// start corner; they are solved by Gaussian elimination without pivoting in ascending
// global index order (DESIGN R-8), redundantly by every box that needs them, so every
// box computes bit-identical values and results do not depend on CTA schedule or GPU
// count.  All values live in global memory; a box also writes the partner values it
// computes (identical bits to what the owner writes).
//
// This is the general path (1D, box shapes outside the specialised engines, the ILU(0)
// factor).  2D 64 x 64 boxes run on sweep2p.cuh / sweep2v.cuh / tri2t.cuh, 3D on
// sweep3.cuh / tri3t.cuh.
#pragma once
#include "common.cuh"

namespace sw {

enum Mode : int { M_FWD = 0, M_T1 = 1, M_T2 = 2, M_FACTOR = 3 };
enum Rhs : int { R_SOR = 0, R_SCALE = 1, R_COEF = 2 };
enum Alpha : int { A_OMEGA_AP = 0, A_INVD = 1 };

struct KParams {
    Geo G;
    int mode, rhs, alpha_mode;
    int base;        // c(k) direction bits for this pass
    int j;           // coupling degree handled by an M_T2 pass
    double omega[8]; // per direction bits
    double coef;     // R_COEF scale
    const double *xold, *src, *b, *invD;
    const double *F[3];
    double *out;
    int *flag;       // bit 0: singular coupled system / ILU pivot
};

__device__ inline bool is_implicit(const Geo &G, int base, const int64_t p[3], int a, int sd) {
    int s = node_bits(G, base, p);
    return sd == (((s >> a) & 1) ? +1 : -1);
}

// dependency: forward p needs q (q implicit for p); transposed p needs q (p implicit for q)
__device__ inline bool depends(const Geo &G, int base, bool transpose, const int64_t p[3], int a, int sd) {
    if (!transpose) return is_implicit(G, base, p, a, sd);
    int64_t q[3] = {p[0], p[1], p[2]};
    q[a] += sd;
    return is_implicit(G, base, q, a, -sd);
}

__device__ inline double node_alpha(const KParams &P, const int64_t g[3]) {
    if (P.alpha_mode == A_INVD) return P.invD[gidx(P.G, g[0], g[1], g[2])];
    int s = node_bits(P.G, P.base, g);
    return P.omega[s] / a_p(P.G, P.F, g);
}

__device__ inline double node_r0(const KParams &P, const int64_t g[3], double alpha) {
    const Geo &G = P.G;
    int64_t i = gidx(G, g[0], g[1], g[2]);
    if (P.rhs == R_SCALE) return alpha * P.src[i];
    if (P.rhs == R_COEF) return P.coef * P.src[i];
    // R_SOR: e = b + sum_{explicit q, axis order} c_pq u_q; r0 = fma(alpha, e, (1-w) u_p)
    int s = node_bits(G, P.base, g);
    double w = P.omega[s];
    double e = P.b[i];
    for (int a = 0; a < G.dim; ++a) {
        int sd = ((s >> a) & 1) ? -1 : +1;
        int64_t q[3] = {g[0], g[1], g[2]};
        q[a] += sd;
        if (in_domain(G, q)) e = fma(face(G, P.F, g, a, sd), P.xold[gidx(G, q[0], q[1], q[2])], e);
    }
    return fma(alpha, e, (1.0 - w) * P.xold[i]);
}

// Solve the coupled set whose members are g with the SCC axes (mask) taking both sides of
// the face at `lo` (lower global coordinate of each pair).  k = 2^popcount(mask) <= 8.
__device__ void solve_set(const KParams &P, bool transpose, const int64_t gl[3], int mask) {
    const Geo &G = P.G;
    int ax[3], na = 0;
    for (int a = 0; a < G.dim; ++a)
        if ((mask >> a) & 1) ax[na++] = a;
    const int k = 1 << na;
    int64_t gm[8][3];
    for (int m = 0; m < k; ++m) {
        gm[m][0] = gl[0]; gm[m][1] = gl[1]; gm[m][2] = gl[2];
        for (int i = 0; i < na; ++i) gm[m][ax[i]] += (m >> i) & 1;
    }
    double M[8][8], rhs[8], u[8];
    for (int p = 0; p < k; ++p) {
        for (int q = 0; q < k; ++q) M[p][q] = (p == q) ? 1.0 : 0.0;
        double al = node_alpha(P, gm[p]);
        double acc = node_r0(P, gm[p], al);
        for (int a = 0; a < G.dim; ++a)
            for (int sd = -1; sd <= 1; sd += 2) {
                int64_t q[3] = {gm[p][0], gm[p][1], gm[p][2]};
                q[a] += sd;
                if (!in_domain(G, q) || !depends(G, P.base, transpose, gm[p], a, sd)) continue;
                double m = al * face(G, P.F, gm[p], a, sd);
                int in = -1;
                if ((mask >> a) & 1) {
                    // partner across the face along a?
                    int bit = -1;
                    for (int i = 0; i < na; ++i)
                        if (ax[i] == a) bit = i;
                    int partner = p ^ (1 << bit);
                    if (gm[partner][a] == q[a]) in = partner;
                }
                if (in >= 0) M[p][in] = -m;
                else acc = fma(m, P.out[gidx(G, q[0], q[1], q[2])], acc);
            }
        rhs[p] = acc;
    }
    if (k == 1) {
        u[0] = rhs[0];
    } else {
        double inv[8];
        for (int p = 0; p < k; ++p) {
            double piv = M[p][p];
            if (!(fabs(piv) >= 1e-14)) atomicOr(P.flag, 1);
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
    }
    for (int m = 0; m < k; ++m) P.out[gidx(G, gm[m][0], gm[m][1], gm[m][2])] = u[m];
}

// D-ILU(0) factor of one node (DESIGN R-C): dd = a_P - sum_{implicit q, same box} c^2 invD_q
__device__ void factor_node(const KParams &P, const int64_t g[3]) {
    const Geo &G = P.G;
    double dd = a_p(G, P.F, g);
    for (int a = 0; a < G.dim; ++a)
        for (int sd = -1; sd <= 1; sd += 2) {
            int64_t q[3] = {g[0], g[1], g[2]};
            q[a] += sd;
            if (!in_domain(G, q) || !is_implicit(G, P.base, g, a, sd)) continue;
            if (q[a] / G.T[a] != g[a] / G.T[a]) continue;   // same box only
            double f = face(G, P.F, g, a, sd);
            double t2 = f * f;
            dd = fma(-t2, P.out[gidx(G, q[0], q[1], q[2])], dd);
        }
    if (!(dd > 0.0)) atomicOr(P.flag, 1);
    P.out[gidx(G, g[0], g[1], g[2])] = 1.0 / dd;
}

template <int DIM>
__global__ void __launch_bounds__(128) k_generic(KParams P) {
    SW_JITTER_POINT();
    const Geo &G = P.G;
    // tile of this CTA (local tile index, x fastest)
    int64_t t = blockIdx.x;
    int64_t R[3] = {0, 0, 0};
    R[0] = t % G.nt[0];
    if (DIM > 1) R[1] = (t / G.nt[0]) % G.nt[1];
    if (DIM > 2) R[2] = t / ((int64_t)G.nt[0] * G.nt[1]);
    int s[3] = {0, 0, 0}, cpl[3] = {0, 0, 0};
    int64_t lo_g[3] = {0, 0, 0};
    for (int a = 0; a < DIM; ++a) {
        R[a] += G.toff[a];
        s[a] = ((P.base >> a) & 1) ^ (int)(R[a] & 1);
        cpl[a] = s[a] ? (R[a] < G.ntg[a] - 1) : (R[a] > 0);
        lo_g[a] = R[a] * G.T[a];
    }
    const bool transpose = (P.mode == M_T1 || P.mode == M_T2);
    const bool ascending = (P.mode == M_FWD || P.mode == M_FACTOR);
    int lo[3] = {0, 0, 0};
    if (P.mode == M_FWD)
        for (int a = 0; a < DIM; ++a) lo[a] = -cpl[a];
    int dmax = 0;
    for (int a = 0; a < DIM; ++a) dmax += G.T[a] - 1;
    int w1 = (DIM > 1) ? G.T[1] - lo[1] : 1;
    int w2 = (DIM > 2) ? G.T[2] - lo[2] : 1;
    int nlines = w1 * w2;
    for (int it = 0; it <= dmax; ++it) {
        int d = ascending ? it : dmax - it;
        for (int line = threadIdx.x; line < nlines; line += blockDim.x) {
            int l[3] = {0, 0, 0};
            if (DIM > 1) l[1] = lo[1] + line % w1;
            if (DIM > 2) l[2] = lo[2] + line / w1;
            int rem = d;
            for (int a = 1; a < DIM; ++a) rem -= (l[a] >= 0) ? l[a] : -1 - l[a];
            if (rem < 0 || rem >= G.T[0]) continue;
            for (int c = 0; c < 2; ++c) {
                if (c == 1 && !(rem == 0 && lo[0] < 0)) break;
                l[0] = (c == 0) ? rem : -1;
                // global coordinates and coupled-set axes of this node
                int64_t g[3] = {0, 0, 0};
                int mask = 0, own = 1;
                for (int a = 0; a < DIM; ++a) {
                    g[a] = s[a] ? (lo_g[a] + G.T[a] - 1 - l[a]) : (lo_g[a] + l[a]);
                    if (cpl[a] && (l[a] == 0 || l[a] == -1)) mask |= 1 << a;
                    if (l[a] < 0) own = 0;
                }
                int deg = __popc(mask);
                if (P.mode == M_FACTOR) { factor_node(P, g); continue; }
                if (P.mode == M_T1) {
                    if (deg == 0) solve_set(P, true, g, 0);
                    continue;
                }
                if (P.mode == M_T2) {
                    if (!own || deg != P.j) continue;
                } else {
                    // forward: the member with the lowest global coordinates leads
                    bool leader = true;
                    for (int a = 0; a < DIM; ++a)
                        if ((mask >> a) & 1) {
                            int64_t other = s[a] ? (lo_g[a] + G.T[a] - 1 - (-1 - l[a])) : (lo_g[a] + (-1 - l[a]));
                            if (other < g[a]) leader = false;
                        }
                    if (!leader) continue;
                }
                // lower corner of the coupled set
                int64_t gl[3] = {g[0], g[1], g[2]};
                for (int a = 0; a < DIM; ++a)
                    if ((mask >> a) & 1) {
                        int64_t other = s[a] ? (lo_g[a] + G.T[a] - 1 - (-1 - l[a])) : (lo_g[a] + (-1 - l[a]));
                        if (other < gl[a]) gl[a] = other;
                    }
                solve_set(P, transpose, gl, mask);
            }
        }
        __syncthreads();
    }
}


}  // namespace sw
