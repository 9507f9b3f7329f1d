// sweep3.cuh -- 3D decomposed SOR sweep and block-triangular solves (7-point stencil), any box
// T0 x T1 x T2 whose window fits in shared memory, sm_100a.
//
// One CTA (4 warps) per box, four CTAs per SM.  Shared memory holds four compact arrays over
// the extended box [-1, T) per axis in LOCAL coordinates (local +a points away from the box's
// start corner): X (r0, then the results, in place) and C0, C1, C2, the coupling alpha c of
// every active node toward its implicit side along x, y, z.  Active nodes are the box's own
// nodes and the partner layers across its coupled start faces (the other members of the coupled
// 2x2 / 4x4 / 8x8 systems), recomputed redundantly by both boxes.
//  1. Prologue (all warps): r0 and the three couplings of every active node (DESIGN R-7) from
//     x_old / src, b / 1/D~ and the faces read straight from global memory (no halo window: the
//     3D halo is 3.4x the box), one branch-free correctly rounded division per node; pair pivots.
//  2. Sets of two or more coupled faces: the 8 x 8 corner by 8 lanes, the 4 x 4 edge chains by
//     one warp each (factored in parallel, substituted in order); Gaussian elimination without
//     pivoting in ascending global index (DESIGN R-8).
//  3. Level loop (warp 0): the x-face sheet, then a branch-free shuffle wavefront in which lane
//     (j, k) owns the x-line and updates node (s - j - k, j, k) at step s; a node on one coupled
//     face solves its 2 x 2 pair with the partner layer.
//  4. Write-back of the box, coalesced along x.
// Same operations and order as the oracle, so the result is bitwise identical to it.
#pragma once
#include <cuda.h>

#include "common.cuh"
#include "sweep2p.cuh"

namespace sw {

namespace k3 {
constexpr int NT = 128;        // threads per CTA
constexpr int MAXLINES = 64;   // T1 * T2
}  // namespace k3

struct Sweep3Args {
    Geo G;
    int base;
    double omega[8];
    const double *xin;          // x_old (SOR) or the solve's source array
    const double *aux;          // b (SOR) or 1/D~ (ILU) or null
    const double *f0, *f1, *f2; // face arrays or null (unit)
    double *out;
    int *flag;
    double coef;
    int tri, invd_mode, rscale, couple;
};

// Solve one coupled set on the axes AXES (K = 2^popcount members) whose own member sits at
// window word w.  Member S (bit t set = across the t-th set axis) is w - sum_t st[ax_t]; in
// ascending global index its rank is S ^ m, m_t = (s_{ax_t} == 0), so the system is built
// directly in rank space with compile-time indices.  Row of member S:
//   u_S - sum_t C_{ax_t}(S) u_{S ^ (1<<t)} = r0_S + sum_{b not in AXES, axis order} C_b(S) u(S - st_b).
template <int AXES>
__device__ __forceinline__ void solve_set3(double *X, int WS, int w, const int st[3], int sbits, int *flag) {
    // couplings of axis a live at X[(a + 1) WS + w] (one shared array: plain LDS addressing)
    constexpr int NA = ((AXES >> 0) & 1) + ((AXES >> 1) & 1) + ((AXES >> 2) & 1);
    constexpr int K = 1 << NA;
    constexpr int A0 = (AXES & 1) ? 0 : ((AXES & 2) ? 1 : 2);
    constexpr int A1 = (NA < 2) ? -1 : ((AXES & 1) ? ((AXES & 2) ? 1 : 2) : 2);
    constexpr int A2 = (NA < 3) ? -1 : 2;
    constexpr int AX[3] = {A0, A1, A2};
    int m = 0;
#pragma unroll
    for (int t = 0; t < NA; ++t) m |= (((sbits >> AX[t]) & 1) == 0) << t;
    double M[K][K], rhs[K], u[K];
    int wi[K];
#pragma unroll
    for (int r = 0; r < K; ++r) {
        const int S = r ^ m;
        int wS = w;
#pragma unroll
        for (int t = 0; t < NA; ++t)
            if ((S >> t) & 1) wS -= st[AX[t]];
        double acc = X[wS];
#pragma unroll
        for (int b = 0; b < 3; ++b)
            if (!((AXES >> b) & 1)) acc = fma(X[(b + 1) * WS + wS], X[wS - st[b]], acc);
        rhs[r] = acc;
        wi[r] = wS;
#pragma unroll
        for (int q = 0; q < K; ++q) M[r][q] = (r == q) ? 1.0 : 0.0;
#pragma unroll
        for (int t = 0; t < NA; ++t) M[r][r ^ (1 << t)] = -X[(AX[t] + 1) * WS + wS];
    }
    ge_solve_k<K>(M, rhs, u, flag);
#pragma unroll
    for (int r = 0; r < K; ++r) X[wi[r]] = u[r];
}

__device__ __forceinline__ double shfl_up_f64(double v, int delta) {   // full warp, converged
    int lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "d"(v));
    asm volatile("shfl.sync.up.b32 %0, %0, %1, 0, 0xffffffff;" : "+r"(lo) : "r"(delta));
    asm volatile("shfl.sync.up.b32 %0, %0, %1, 0, 0xffffffff;" : "+r"(hi) : "r"(delta));
    double r;
    asm("mov.b64 %0, {%1, %2};" : "=d"(r) : "r"(lo), "r"(hi));
    return r;
}

// A 4-member set (an edge of two coupled faces) split into the part that depends only on the
// couplings (the elimination of the matrix: multipliers, eliminated upper triangle, reciprocal
// pivots) and the part that depends on the chain (right-hand side, its elimination, back
// substitution).  The operations and their order are exactly those of ge_solve_k<4>, so the
// result is the same bit for bit; the split lets every set of an edge be factored in parallel.
struct Fac4 {
    double l[6], U[6], inv[4];
};

template <int AXES>
__device__ __forceinline__ void factor4(const double *X, int WS, int w, const int st[3], int sbits, Fac4 &F,
                                        int &fl) {
    constexpr int A0 = (AXES & 1) ? 0 : 1;
    constexpr int A1 = (AXES & 4) ? 2 : 1;
    constexpr int AX[2] = {A0, A1};
    int m = 0;
#pragma unroll
    for (int t = 0; t < 2; ++t) m |= (((sbits >> AX[t]) & 1) == 0) << t;
    double M[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int S = r ^ m;
        int wS = w;
#pragma unroll
        for (int t = 0; t < 2; ++t)
            if ((S >> t) & 1) wS -= st[AX[t]];
#pragma unroll
        for (int q = 0; q < 4; ++q) M[r][q] = (r == q) ? 1.0 : 0.0;
#pragma unroll
        for (int t = 0; t < 2; ++t) M[r][r ^ (1 << t)] = -X[(AX[t] + 1) * WS + wS];
    }
    int li = 0;
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        const double piv = M[p][p];
        fl |= !(fabs(piv) >= 1e-14);
        F.inv[p] = div_rn(1.0, piv);
#pragma unroll
        for (int q = p + 1; q < 4; ++q) {
            const double l = M[q][p] * F.inv[p];
            F.l[li++] = l;
#pragma unroll
            for (int j = p + 1; j < 4; ++j) M[q][j] = fma(-l, M[p][j], M[q][j]);
        }
    }
    int ui = 0;
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int j = p + 1; j < 4; ++j) F.U[ui++] = M[p][j];
}

template <int AXES>
__device__ __forceinline__ void subst4(double *X, int WS, int w, const int st[3], int sbits, const Fac4 &F) {
    constexpr int A0 = (AXES & 1) ? 0 : 1;
    constexpr int A1 = (AXES & 4) ? 2 : 1;
    constexpr int AX[2] = {A0, A1};
    constexpr int B = 3 - A0 - A1;            // the chain axis
    int m = 0;
#pragma unroll
    for (int t = 0; t < 2; ++t) m |= (((sbits >> AX[t]) & 1) == 0) << t;
    double rhs[4], u[4];
    int wi[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int S = r ^ m;
        int wS = w;
#pragma unroll
        for (int t = 0; t < 2; ++t)
            if ((S >> t) & 1) wS -= st[AX[t]];
        rhs[r] = fma(X[(B + 1) * WS + wS], X[wS - st[B]], X[wS]);
        wi[r] = wS;
    }
    int li = 0;
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = p + 1; q < 4; ++q) {
            rhs[q] = fma(-F.l[li], rhs[p], rhs[q]);
            ++li;
        }
    constexpr int UI[4] = {0, 3, 5, 6};       // first U entry of row p
#pragma unroll
    for (int p = 3; p >= 0; --p) {
        double sacc = rhs[p];
#pragma unroll
        for (int j = p + 1; j < 4; ++j) sacc = fma(-F.U[UI[p] + (j - p - 1)], u[j], sacc);
        u[p] = sacc * F.inv[p];
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) X[wi[r]] = u[r];
}

// The corner set of three coupled faces (8 members), eliminated by lanes 0..7 of one warp (lane
// q owns row q; step p: every lane below p updates its row) in a shared scratch of >= 80
// doubles; the same operations in the same order as ge_solve_k<8>, then lane 0 back-substitutes.
__device__ __forceinline__ void corner8_coop(double *X, int WS, double *scr, int lane, int w, const int st[3], int sbits,
                                             int *flag) {
    double *M = scr, *rhs = scr + 64, *inv = scr + 72;
    int m = 0;
#pragma unroll
    for (int t = 0; t < 3; ++t) m |= (((sbits >> t) & 1) == 0) << t;
    int wS = w;
    if (lane < 8) {
        const int r = lane, S = r ^ m;
#pragma unroll
        for (int t = 0; t < 3; ++t)
            if ((S >> t) & 1) wS -= st[t];
#pragma unroll
        for (int q = 0; q < 8; ++q) M[r * 8 + q] = (r == q) ? 1.0 : 0.0;
#pragma unroll
        for (int t = 0; t < 3; ++t) M[r * 8 + (r ^ (1 << t))] = -X[(t + 1) * WS + wS];
        rhs[r] = X[wS];
    }
    __syncwarp();
    for (int p = 0; p < 8; ++p) {
        const double piv = M[p * 8 + p];
        const double ip = div_rn(1.0, piv);
        if (lane == 0) {
            inv[p] = ip;
            if (!(fabs(piv) >= 1e-14)) atomicOr(flag, 1);
        }
        if (lane > p && lane < 8) {
            const double l = M[lane * 8 + p] * ip;
            for (int j = p + 1; j < 8; ++j) M[lane * 8 + j] = fma(-l, M[p * 8 + j], M[lane * 8 + j]);
            rhs[lane] = fma(-l, rhs[p], rhs[lane]);
        }
        __syncwarp();
    }
    if (lane == 0) {
        double u[8];
#pragma unroll
        for (int p = 7; p >= 0; --p) {
            double sacc = rhs[p];
#pragma unroll
            for (int j = p + 1; j < 8; ++j) sacc = fma(-M[p * 8 + j], u[j], sacc);
            u[p] = sacc * inv[p];
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) rhs[r] = u[r];
    }
    __syncwarp();
    if (lane < 8) X[wS] = rhs[lane];
    __syncwarp();
}

// one edge chain: lane t-1 of the calling warp owns set t (t = 1 .. T-1 <= 32); every lane
// factors its set while the corner is being solved, then the sets are substituted in order
template <int AXES>
__device__ __forceinline__ void edge_chain(double *X, int WS, int lane, int T, int w1, int step, const int st[3],
                                           int sbits, int *flag, bool run) {
    Fac4 F;
    int fl = 0;
    const bool mine = run && lane + 1 < T;
    if (mine) factor4<AXES>(X, WS, w1 + lane * step, st, sbits, F, fl);
    if (fl) atomicOr(flag, 1);
    __syncthreads();                          // the corner set is in place
    if (run)
        for (int t = 1; t < T; ++t) {
            if (lane == t - 1) subst4<AXES>(X, WS, w1 + (t - 1) * step, st, sbits, F);
            __syncwarp();
        }
}

#ifdef SW_DEBUG3
__device__ double sw_dbg3[4 * 8192];
__device__ int sw_dbg3_block = -1;
#endif

template <bool FACES>
__global__ void __launch_bounds__(k3::NT, 4) k_sweep3(Sweep3Args A) {
    extern __shared__ __align__(128) double sm[];
    const Geo &G = A.G;
    const int T0 = G.T[0], T1 = G.T[1], T2 = G.T[2];
    // compact arrays over the extended box [-1, T) per axis in LOCAL coordinates (sweep order:
    // local +a points away from the box's start corner), so every step below is positive
    const int E0 = T0 + 1, E1 = T1 + 1, E2 = T2 + 1;
    const int WS = E0 * E1 * E2;
    double *const X = sm;                               // r0 of the active nodes, then their results
    double *const C0 = sm + WS, *const C1 = sm + 2 * WS, *const C2 = sm + 3 * WS;
    double *const PV = sm + 4 * WS;                     // pair pivots: y-face sheet [T2][T0], z-face [T1][T0]
    double *const SCR = PV + T0 * (T1 + T2);            // corner elimination scratch (80 doubles)
    auto CC = [&](int a, int w) -> double & { return sm[(a + 1) * WS + w]; };   // coupling of axis a
    const int tid = threadIdx.x;
    // box, direction bits, coupled start faces
    const int tx = blockIdx.x % G.nt[0];
    const int ty = (blockIdx.x / G.nt[0]) % G.nt[1];
    const int tz = blockIdx.x / (G.nt[0] * G.nt[1]);
    const int64_t R[3] = {tx, ty, tz + G.toff[2]};
    int sb = 0, cb = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const int s = ((A.base >> a) & 1) ^ (int)(R[a] & 1);
        const bool c = A.couple && (s ? (R[a] < G.ntg[a] - 1) : (R[a] > 0));
        sb |= s << a;
        cb |= (int)c << a;
    }
    const int st[3] = {1, E0, E0 * E1};               // compact step of local +a
    auto wof = [&](int l0, int l1, int l2) { return (l0 + 1) + E0 * ((l1 + 1) + E1 * (l2 + 1)); };
    const int64_t P0 = G.P0, P01 = G.P01;
    const int64_t gbase = (int64_t)tz * T2 * P01 + (int64_t)ty * T1 * P0 + (int64_t)tx * T0;   // padded (box min - 2)
    const int64_t Sg[3] = {1, P0, P01};

    SW_TMARK(t_start);
    // ---------------------------------------------------------------- 1. prologue
    // Every node of the extended box: r0 and the couplings alpha c toward its implicit side of the
    // active nodes (own nodes and the partner layers across coupled start faces, DESIGN R-7), zero
    // for the rest (the layers across uncoupled faces are read only through zero couplings).
    // x_old / src, b / 1/D~ and the faces come straight from global memory (L1/L2: neighbouring
    // boxes share their halos), coalesced along x; the loop walks e = (l0, l1, l2) in mixed radix.
    {
        const double *__restrict__ xin = A.xin;
        const double *__restrict__ aux = A.aux;
        const double *__restrict__ F0 = A.f0, *__restrict__ F1 = A.f1, *__restrict__ F2 = A.f2;
        int l0 = tid % E0, l1 = (tid / E0) % E1, l2 = tid / (E0 * E1);
        const int a0 = k3::NT % E0, a1 = (k3::NT / E0) % E1, a2 = k3::NT / (E0 * E1);
        const bool need_x = !A.tri, need_aux = !A.tri || A.invd_mode;
        constexpr int KB = 3;      // nodes per batch: all their loads are issued before any use
        for (int e0 = tid; e0 < WS; e0 += KB * k3::NT) {
            int lvv[KB][3], Lm[KB];
            bool on[KB];
            int64_t gg[KB];
#pragma unroll
            for (int kb = 0; kb < KB; ++kb) {
                lvv[kb][0] = l0 - 1; lvv[kb][1] = l1 - 1; lvv[kb][2] = l2 - 1;
                const int L = (l0 < 1 ? 1 : 0) | (l1 < 1 ? 2 : 0) | (l2 < 1 ? 4 : 0);
                Lm[kb] = L;
                on[kb] = l2 < E2 && (L & cb) == L;
                const int w0 = 2 + (((sb >> 0) & 1) ? T0 - 1 - lvv[kb][0] : lvv[kb][0]);
                const int w1 = 2 + (((sb >> 1) & 1) ? T1 - 1 - lvv[kb][1] : lvv[kb][1]);
                const int w2 = 2 + (((sb >> 2) & 1) ? T2 - 1 - lvv[kb][2] : lvv[kb][2]);
                // inactive nodes load from the box's first node (always inside the padded array)
                gg[kb] = on[kb] ? gbase + w0 + (int64_t)w1 * P0 + (int64_t)w2 * P01 : gbase + 2 + 2 * P0 + 2 * P01;
                l0 += a0;
                const int c0 = l0 >= E0;
                l0 -= c0 ? E0 : 0;
                l1 += a1 + c0;
                const int c1 = l1 >= E1;
                l1 -= c1 ? E1 : 0;
                l2 += a2 + c1;
            }
            double f[KB][3][2], xn[KB][3], xo[KB], av[KB];
#pragma unroll
            for (int kb = 0; kb < KB; ++kb) {
                const int64_t g = gg[kb];
                if (FACES) {
                    f[kb][0][0] = __ldg(F0 + g); f[kb][0][1] = __ldg(F0 + g + 1);
                    f[kb][1][0] = __ldg(F1 + g); f[kb][1][1] = __ldg(F1 + g + P0);
                    f[kb][2][0] = __ldg(F2 + g); f[kb][2][1] = __ldg(F2 + g + P01);
                } else {
#pragma unroll
                    for (int a = 0; a < 3; ++a) f[kb][a][0] = f[kb][a][1] = 1.0;
                }
                xo[kb] = __ldg(xin + g);
                av[kb] = need_aux ? __ldg(aux + g) : 0.0;
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    const bool hi = (((Lm[kb] >> a) & 1) != 0) != (((sb >> a) & 1) != 0);   // implicit side is global +a
                    xn[kb][a] = need_x ? __ldg(xin + (hi ? g - Sg[a] : g + Sg[a])) : 0.0;
                }
            }
#pragma unroll
            for (int kb = 0; kb < KB; ++kb) {
                const int e = e0 + kb * k3::NT;
                if (e >= WS) break;
                const int L = Lm[kb];
                double r0 = 0.0, c[3] = {0.0, 0.0, 0.0};
                if (on[kb]) {
                    const double(&fk)[3][2] = f[kb];
                    const double ap = (((fk[0][0] + fk[0][1]) + (fk[1][0] + fk[1][1])) + (fk[2][0] + fk[2][1])) + G.beta;
                    bool hi[3];
#pragma unroll
                    for (int a = 0; a < 3; ++a) hi[a] = (((L >> a) & 1) != 0) != (((sb >> a) & 1) != 0);
                    double al;
                    if (!A.tri) {
                        const double w_ = A.omega[sb ^ L];             // the node's own box's direction bits
                        al = div_rn(w_, ap);
                        double ev = av[kb];
#pragma unroll
                        for (int a = 0; a < 3; ++a) ev = fma(hi[a] ? fk[a][0] : fk[a][1], xn[kb][a], ev);
                        r0 = fma(al, ev, (1.0 - w_) * xo[kb]);
                    } else {
                        al = A.invd_mode ? av[kb] : div_rn(A.omega[0], ap);
                        r0 = A.rscale ? al * xo[kb] : A.coef * xo[kb];
                    }
#pragma unroll
                    for (int a = 0; a < 3; ++a) {
                        // no coupling across an uncoupled start face: the oracle omits the term (physical
                        // boundary) and the first pass of the transposed solve must not see the neighbour box
                        const bool cut = !((L >> a) & 1) && lvv[kb][a] == 0 && !((cb >> a) & 1);
                        c[a] = cut ? 0.0 : al * (hi[a] ? fk[a][1] : fk[a][0]);
                    }
                }
                X[e] = r0;
                C0[e] = c[0];
                C1[e] = c[1];
                C2[e] = c[2];
            }
        }
    }
    SW_TMARK(t_pro_own);
    SW_TADD(8, t_start, t_pro_own);
    __syncthreads();
    // pivots 1 / (1 - m m') of the face pairs that the level loop solves (y- and z-face sheets)
    const bool fast_lines = T1 * T2 <= 32;
    if (fast_lines) {
        const int ny = ((cb & 2) ? T0 * T2 : 0), nz = ((cb & 4) ? T0 * T1 : 0);
        int fl = 0;
        for (int e = tid; e < ny + nz; e += k3::NT) {
            int i, j, k, a, pi;
            if (e < ny) { i = e % T0; k = e / T0; j = 0; a = 1; pi = e; }
            else { i = (e - ny) % T0; j = (e - ny) / T0; k = 0; a = 2; pi = T0 * T2 + (e - ny); }
            const int m = (i == 0 ? (cb & 1) : 0) | (j == 0 ? (cb & 2) : 0) | (k == 0 ? (cb & 4) : 0);
            if (__popc(m) != 1) continue;                         // sets of two or more faces: step 3
            const int w = wof(i, j, k), q = w - st[a];
            const double m11 = fma(CC(a, w), -CC(a, q), 1.0);
            fl |= !(fabs(m11) >= 1e-14);
            PV[pi] = div_rn(1.0, m11);
        }
        if (fl) atomicOr(A.flag, 1);
        __syncthreads();
    }
    SW_TMARK(t_prologue);
    const int lt = tid;
    // ---------------------------------------------------------------- 2. corner and edge sets
    const int ncpl = __popc(cb);
    if (ncpl >= 2) {
        if (cb == 7) {
            if (lt < 32) corner8_coop(X, WS, SCR, lt, wof(0, 0, 0), st, sb, A.flag);
        } else if (lt == 0) {
            const int w = wof(0, 0, 0);
            switch (cb) {
                case 3: solve_set3<3>(X, WS, w, st, sb, A.flag); break;
                case 5: solve_set3<5>(X, WS, w, st, sb, A.flag); break;
                default: solve_set3<6>(X, WS, w, st, sb, A.flag); break;
            }
        }
        SW_TMARK(t_corner);
        SW_TADDT(12, t_prologue, t_corner, 0);
        // the edge chains (independent of each other), one per warp: x-edge in warp 1, y-edge in
        // warp 2, z-edge in warp 3 (factored in parallel with the corner, substituted in order)
        const int warp = lt >> 5, lane = lt & 31;
        if (warp == 1) edge_chain<6>(X, WS, lane, T0, wof(1, 0, 0), st[0], st, sb, A.flag, (cb & 6) == 6);
        else if (warp == 2) edge_chain<5>(X, WS, lane, T1, wof(0, 1, 0), st[1], st, sb, A.flag, (cb & 5) == 5);
        else if (warp == 3) edge_chain<3>(X, WS, lane, T2, wof(0, 0, 1), st[2], st, sb, A.flag, (cb & 3) == 3);
        else __syncthreads();
        __syncthreads();
    }

#ifdef SW_DEBUG3
    if ((int)blockIdx.x == sw_dbg3_block)
        for (int i = tid; i < WS; i += k3::NT) {
            sw_dbg3[i] = X[i];
            sw_dbg3[8192 + i] = C0[i];
        }
#endif
    SW_TMARK(t_sets);
    // ---------------------------------------------------------------- 3. level loop (warp 0)
    if (fast_lines) {
        // (a) the x-face sheet (pairs (0, j, k) / (-1, j, k)), a 2D recurrence over (j, k)
        if (lt < 32 && (cb & 1)) {
            const int j = lt % T1, k = lt / T1;
            const bool on = lt < T1 * T2;
            const int m = 1 | (j == 0 ? (cb & 2) : 0) | (k == 0 ? (cb & 4) : 0);
            const int w = on ? wof(0, j, k) : 0, q = w - st[0];
            int fl = 0;
            for (int d = 0; d <= T1 + T2 - 2; ++d) {
                if (on && j + k == d && m == 1) {
                    const double rp = fma(CC(2, w), X[w - st[2]], fma(CC(1, w), X[w - st[1]], X[w]));
                    const double rq = fma(CC(2, q), X[q - st[2]], fma(CC(1, q), X[q - st[1]], X[q]));
                    const bool qfirst = (sb & 1) == 0;
                    const double ra = qfirst ? rq : rp, rb = qfirst ? rp : rq;
                    const double cw = CC(0, w), cq = CC(0, q);
                    const double mab = qfirst ? cq : cw, mba = qfirst ? cw : cq;
                    const double m11 = fma(mba, -mab, 1.0);
                    fl |= !(fabs(m11) >= 1e-14);
                    const double ub = fma(mba, ra, rb) * div_rn(1.0, m11);
                    const double ua = fma(mab, ub, ra) * 1.0;
                    X[w] = qfirst ? ub : ua;
                    X[q] = qfirst ? ua : ub;
                }
                __syncwarp();
            }
            if (fl) atomicOr(A.flag, 1);
        }
        SW_TMARK(t_xs);
        SW_TADDT(13, t_sets, t_xs, 0);
        // (b) all other nodes: lane (j, k) owns the x-line and updates node i = s - j - k at step
        //     s; S and B arrive from lanes l-1 and l-T1 by shuffles, and so do the partner values
        //     of the y- and z-face sheets (which each lane on such a face carries in registers).
        //     One branch-free instruction stream for every kind of lane: a plain lane is a "pair"
        //     with zero couplings and unit pivot, which leaves its node formula exact; the x-edge
        //     lane (solved in step 2) only reloads and forwards its values.
        if (lt < 32) {
            const int lane = lt, nl = T1 * T2;
            const bool on = lane < nl;
            const int j = on ? lane % T1 : 0, k = on ? lane / T1 : 0;
            const bool yc = j == 0 && (cb & 2), zc = k == 0 && (cb & 4);
            const bool edge = yc && zc, ypair = yc && !zc, zpair = zc && !yc, pair = ypair || zpair;
            const int i0 = (cb & 1) ? 1 : 0;
            const int sx = st[0], sy = st[1], sz = st[2];
            const int sa = ypair ? sy : (zpair ? sz : 0);                 // step toward the pair partner
            const int wl = wof(0, j, k);
            const int pvb = ypair ? T0 * k : T0 * T2 + T0 * j;           // pivots of the lane's pairs
            const bool qf = pair ? (((sb >> (ypair ? 1 : 2)) & 1) == 0) : true;   // partner first in index order
            // addresses of the other transverse coupling of the partner: z for y-pairs, y for z-pairs
            const int oq_arr = ypair ? 3 : 2;                             // (axis + 1) of that coupling
            const int pa_arr = ypair ? 2 : 3;                             // (axis + 1) of the pair coupling
            double W = i0 ? X[wl] : 0.0;
            double Wq = (i0 && pair) ? X[wl - sa] : 0.0;                 // partner value at i0 - 1
            double u = 0.0, py = 0.0, pz = 0.0;
            const int NS = T0 + T1 + T2 - 2;
            auto ld = [&](int s, double (&v)[11]) {
                int i = s - j - k;
                i = i < 0 ? 0 : (i >= T0 ? T0 - 1 : i);                   // clamp idle lanes' addresses
                const int w = wl + i * sx, q = pair ? w - sa : w;
                v[0] = X[w];                    // r0 (edge lane: its solved value)
                v[1] = sm[WS + w];              // C_x
                v[2] = sm[2 * WS + w];          // C_y
                v[3] = sm[3 * WS + w];          // C_z
                v[4] = X[q];                    // partner r0
                v[5] = sm[WS + q];              // partner C_x
                v[6] = sm[oq_arr * WS + q];     // partner other transverse coupling
                v[7] = sm[pa_arr * WS + q];     // partner pair coupling
                v[8] = pair ? PV[pvb + i] : 1.0;  // pivot inverse (prologue)
                v[9] = edge ? X[w - sy] : 0.0;  // edge: its y-partner value
                v[10] = edge ? X[w - sz] : 0.0; //       its z-partner value
            };
            double nv[11];
            ld(0, nv);
            for (int s = 0; s < NS; ++s) {
                const double Sv = shfl_up_f64(u, 1), Bv = shfl_up_f64(u, T1);
                const double Sq = shfl_up_f64(pz, 1), Bq = shfl_up_f64(py, T1);
                double v[11];
#pragma unroll
                for (int t = 0; t < 11; ++t) v[t] = nv[t];
                if (s + 1 < NS) ld(s + 1, nv);
                const int i = s - j - k;
                const bool act = on && i >= i0 && i < T0;
                const int w = wl + (i < 0 ? 0 : (i >= T0 ? T0 - 1 : i)) * sx;
                // own row: x, y (unless the y pair), z (unless the z pair), in axis order
                const double cyE = ypair ? 0.0 : v[2], czE = zpair ? 0.0 : v[3];
                const double rp = fma(czE, Bv, fma(cyE, Sv, fma(v[1], W, v[0])));
                // partner row: x, then the other transverse axis
                const double Oq = ypair ? Bq : Sq;
                const double rq = fma(pair ? v[6] : 0.0, Oq, fma(pair ? v[5] : 0.0, Wq, v[4]));
                const double cw = ypair ? v[2] : (zpair ? v[3] : 0.0), cq = pair ? v[7] : 0.0;
                const double ra = qf ? rq : rp, rb = qf ? rp : rq;
                const double mab = qf ? cq : cw, mba = qf ? cw : cq;
                const double ub = fma(mba, ra, rb) * v[8];
                const double ua = fma(mab, ub, ra) * 1.0;
                double un = qf ? ub : ua;
                const double pv = qf ? ua : ub;
                un = edge ? v[0] : un;
                st_shared_if(X + w, un, act && !edge);
                u = sel_f64(act, un, u);
                W = sel_f64(act, un, W);              // idle (joining) lanes keep W = value at i0 - 1
                Wq = sel_f64(act && pair, pv, Wq);
                py = sel_f64(act, ypair ? pv : (edge ? v[9] : py), py);
                pz = sel_f64(act, zpair ? pv : (edge ? v[10] : pz), pz);
            }
            SW_TMARK(t_wf);
            SW_TADDT(9, t_xs, t_wf, 0);
        }
    } else if (lt < 32) {
        const int nl = T1 * T2, nlev = T0 + T1 + T2 - 2;
        // per-lane lines (at most two): offset j + k of the level, word of node i = 0, coupled-face
        // mask of the line (y-face if j == 0, z-face if k == 0)
        int jk[2], wl[2], lm[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int ln = lt + 32 * h;
            const int j = ln % T1, k = ln / T1;
            jk[h] = (ln < nl) ? j + k : (1 << 20);          // never active
            wl[h] = wof(0, ln < nl ? j : 0, ln < nl ? k : 0);
            lm[h] = (j == 0 ? (cb & 2) : 0) | (k == 0 ? (cb & 4) : 0);
        }
        const int s0 = st[0], st0 = st[0], st1 = st[1], st2 = st[2];
        int fl = 0;
        for (int d = 0; d < nlev; ++d) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int i = d - jk[h];
                if (i < 0 || i >= T0) continue;
                const int m = (i == 0 ? (cb & 1) : 0) | lm[h];
                const int w = wl[h] + i * s0;
                if (m == 0) {
                    double acc = X[w];
                    acc = fma(C0[w], X[w - st0], acc);
                    acc = fma(C1[w], X[w - st1], acc);
                    acc = fma(C2[w], X[w - st2], acc);
                    X[w] = acc;
                } else if ((m & (m - 1)) == 0) {               // one coupled face: 2 x 2 pair
                    const int a = (m & 1) ? 0 : ((m & 2) ? 1 : 2);
                    const int sta = (m & 1) ? st0 : ((m & 2) ? st1 : st2);
                    const int q = w - sta;
                    double rp = X[w], rq = X[q];
                    // the two axes other than a, in axis order
                    const int b1 = (a == 0) ? 1 : 0, b2 = (a == 2) ? 1 : 2;
                    const int s1 = (a == 0) ? st1 : st0, s2 = (a == 2) ? st1 : st2;
                    rp = fma(CC(b1, w), X[w - s1], rp);
                    rq = fma(CC(b1, q), X[q - s1], rq);
                    rp = fma(CC(b2, w), X[w - s2], rp);
                    rq = fma(CC(b2, q), X[q - s2], rq);
                    const bool qfirst = ((sb >> a) & 1) == 0;   // partner has the lower global index
                    const double ra = qfirst ? rq : rp, rb = qfirst ? rp : rq;
                    const double cw = CC(a, w), cq = CC(a, q);
                    const double mab = qfirst ? cq : cw, mba = qfirst ? cw : cq;
                    const double m11 = fma(mba, -mab, 1.0);
                    fl |= !(fabs(m11) >= 1e-14);
                    const double ub = fma(mba, ra, rb) * div_rn(1.0, m11);
                    const double ua = fma(mab, ub, ra) * 1.0;
                    X[w] = qfirst ? ub : ua;
                    X[q] = qfirst ? ua : ub;
                }
                // (sets on two or three faces were solved in step 2)
            }
            __syncwarp();
        }
        if (fl) atomicOr(A.flag, 1);
    }
    __syncthreads();
    SW_TMARK(t_levels);

    // ---------------------------------------------------------------- 4. write-back of the box
    {
        const int n = T0 * T1 * T2;
        int l0 = tid % T0, l1 = (tid / T0) % T1, l2 = tid / (T0 * T1);
        const int a0 = k3::NT % T0, a1 = (k3::NT / T0) % T1, a2 = k3::NT / (T0 * T1);
        for (int e = tid; e < n; e += k3::NT) {
            const int w0 = 2 + (((sb >> 0) & 1) ? T0 - 1 - l0 : l0);
            const int w1 = 2 + (((sb >> 1) & 1) ? T1 - 1 - l1 : l1);
            const int w2 = 2 + (((sb >> 2) & 1) ? T2 - 1 - l2 : l2);
            A.out[gbase + w0 + (int64_t)w1 * P0 + (int64_t)w2 * P01] = X[wof(l0, l1, l2)];
            l0 += a0;
            const int c0 = l0 >= T0;
            l0 -= c0 ? T0 : 0;
            l1 += a1 + c0;
            const int c1 = l1 >= T1;
            l1 -= c1 ? T1 : 0;
            l2 += a2 + c1;
        }
    }
    SW_TMARK(t_end);
    SW_TADD(1, t_start, t_prologue);
    SW_TADD(2, t_prologue, t_sets);
    SW_TADD(3, t_sets, t_levels);
    SW_TADD(4, t_levels, t_end);
    SW_TADD(5, 0, 1);
}

inline size_t sweep3_smem(const Geo &G) {
    const size_t ws = (size_t)(G.T[0] + 1) * (G.T[1] + 1) * (G.T[2] + 1);
    return sizeof(double) * (4 * ws + (size_t)G.T[0] * (G.T[1] + G.T[2]) + 80);
}

// the fast 3D path handles boxes whose compact arrays fit in shared memory
inline bool sweep3_supported(const Geo &G) {
    if (G.dim != 3) return false;
    return (G.T[0] % 2 == 0) && sweep3_smem(G) <= 227 * 1024 && G.T[1] * G.T[2] <= k3::MAXLINES &&
           G.T[0] <= 33 && G.T[1] <= 33 && G.T[2] <= 33 && G.off[0] == 0 && G.off[1] == 0;
}

inline cudaError_t launch_sweep3(const Sweep3Args &A, cudaStream_t s) {
    const size_t smem = sweep3_smem(A.G);
    const bool faces = A.f0 != nullptr;
    if (faces) cudaFuncSetAttribute(k_sweep3<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    else cudaFuncSetAttribute(k_sweep3<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const unsigned tiles = (unsigned)((int64_t)A.G.nt[0] * A.G.nt[1] * A.G.nt[2]);
    if (faces) k_sweep3<true><<<tiles, k3::NT, smem, s>>>(A);
    else k_sweep3<false><<<tiles, k3::NT, smem, s>>>(A);
    return cudaGetLastError();
}

}  // namespace sw
