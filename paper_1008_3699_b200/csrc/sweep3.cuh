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
    int RS, PS;                 // compact-array strides of local +y and +z (host: sweep3_layout)
};

// Compile-time box shapes: SHAPE 1 = 32 x 8 x 4 (config 5), SHAPE 0 = any box (runtime values).
template <int SHAPE>
struct Shape3 {
    __device__ static int t0(const Sweep3Args &A) { return A.G.T[0]; }
    __device__ static int t1(const Sweep3Args &A) { return A.G.T[1]; }
    __device__ static int t2(const Sweep3Args &A) { return A.G.T[2]; }
    __device__ static int rs(const Sweep3Args &A) { return A.RS; }
    __device__ static int ps(const Sweep3Args &A) { return A.PS; }
};
template <>
struct Shape3<1> {
    __device__ static constexpr int t0(const Sweep3Args &) { return 32; }
    __device__ static constexpr int t1(const Sweep3Args &) { return 8; }
    __device__ static constexpr int t2(const Sweep3Args &) { return 4; }
    __device__ static constexpr int rs(const Sweep3Args &) { return 34; }
    __device__ static constexpr int ps(const Sweep3Args &) { return 307; }
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
                                           int sbits, int *flag, bool run, int *done = nullptr) {
    Fac4 F;
    int fl = 0;
    const bool mine = run && lane + 1 < T;
    if (mine) factor4<AXES>(X, WS, w1 + lane * step, st, sbits, F, fl);
    if (fl) atomicOr(flag, 1);
    __syncthreads();                          // the corner set is in place
    if (run)
        for (int t = 1; t < T; ++t) {
            if (lane == t - 1) {
                subst4<AXES>(X, WS, w1 + (t - 1) * step, st, sbits, F);
                if (done)                     // publish: set t is in place (read by the wavefront warp)
                    asm volatile("st.release.cta.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(done)), "r"(t) : "memory");
            }
            __syncwarp();
        }
}


#ifndef SW_KB
#define SW_KB 2
#endif
template <bool FACES, int SHAPE>
__global__ void __launch_bounds__(k3::NT, 4) k_sweep3(Sweep3Args A) {
    extern __shared__ __align__(128) double sm[];
    SW_JITTER_POINT();
    const Geo &G = A.G;
    using SH = Shape3<SHAPE>;
    const int T0 = SH::t0(A), T1 = SH::t1(A), T2 = SH::t2(A);
    // compact arrays over the extended box [-1, T) per axis in LOCAL coordinates (sweep order:
    // local +a points away from the box's start corner), so every step below is positive; the
    // y / z strides RS / PS are padded so that the wavefront's 32 lanes hit distinct banks
    const int E0 = T0 + 1, E1 = T1 + 1, E2 = T2 + 1;
    const int RS = SH::rs(A), PS = SH::ps(A);
    const int WS = PS * E2;
    double *const X = sm;                               // r0 of the active nodes, then their results
    double *const C0 = sm + WS, *const C1 = sm + 2 * WS, *const C2 = sm + 3 * WS;
    // pair data of the 2 x 2 face pairs, a = the member of lower global index: x-face sheet
    // (1 / pivot, m_ab, m_ba) [k][j]; y-face sheet (m_ab, m_ba) [k][i], z-face sheet [j][i] (line
    // stride T0 + 1); then (0, 0) for the lanes without a pair
    double *const PVX = sm + 4 * WS;
    double *const PVY = PVX + 3 * T1 * T2;
    double *const PVZ = PVY + 2 * (T0 + 1) * T2;
    double *const PV1 = PVZ + 2 * (T0 + 1) * T1;
    double *const SCR = PV1 + 4;                        // corner elimination scratch (80 doubles)
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
    const int st[3] = {1, RS, PS};                      // compact step of local +a
    auto wof = [&](int l0, int l1, int l2) { return (l0 + 1) + RS * (l1 + 1) + PS * (l2 + 1); };
    const int64_t P0 = G.P0, P01 = G.P01;
    const int64_t gbase = (int64_t)tz * T2 * P01 + (int64_t)ty * T1 * P0 + (int64_t)tx * T0;   // padded (box min - 2)
    const int64_t Sg[3] = {1, P0, P01};

    SW_TMARK(t_start);
    // ---------------------------------------------------------------- 1. prologue
    // Every node of the extended box: r0 and the couplings alpha c toward its implicit side of the
    // active nodes (own nodes and the partner layers across coupled start faces, DESIGN R-7), zero
    // for the rest (the layers across uncoupled faces and the padding are read only through zero
    // couplings).  x_old / src, b / 1/D~ and the faces come straight from global memory (L1/L2:
    // neighbouring boxes share their halos), coalesced along x, addressed by 32-bit offsets from
    // the box's base: local (m0, m1, m2) sits at o = O0 + m0 d0 + m1 d1 + m2 d2.
    {
        const int P0i = (int)P0, P01i = (int)P01;
        const int Sgi[3] = {1, P0i, P01i};
        int O0 = 0, d[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const int Ta = a == 0 ? T0 : (a == 1 ? T1 : T2);
            const bool sa_ = (sb >> a) & 1;
            O0 += (2 + (sa_ ? Ta - 1 : 0)) * Sgi[a];
            d[a] = sa_ ? -Sgi[a] : Sgi[a];
        }
        const double *__restrict__ xb = A.xin + gbase;
        const double *__restrict__ ab = (A.aux ? A.aux : A.xin) + gbase;
        const double *__restrict__ f0b = (FACES ? A.f0 : A.xin) + gbase;
        const double *__restrict__ f1b = (FACES ? A.f1 : A.xin) + gbase;
        const double *__restrict__ f2b = (FACES ? A.f2 : A.xin) + gbase;
        const bool need_x = !A.tri, need_aux = !A.tri || A.invd_mode;
        // Row-wise: a warp takes a row (local y, z) of the extended box and its lanes consecutive
        // local x, so every address is the row's base plus the lane (one coalesced run per load)
        // and the active / implicit-side / omega choices are row-uniform.  The column at local
        // x = -1 (the partner layer across the x start face) is one extra node per row.
        struct In {
            double f[3][2], xn[3], xo, av;
        };
        auto load = [&](bool on, int o, int L, In &v) {
            if (!on) return;
            if (FACES) {
                v.f[0][0] = __ldg(f0b + o); v.f[0][1] = __ldg(f0b + o + 1);
                v.f[1][0] = __ldg(f1b + o); v.f[1][1] = __ldg(f1b + o + P0i);
                v.f[2][0] = __ldg(f2b + o); v.f[2][1] = __ldg(f2b + o + P01i);
            } else {
#pragma unroll
                for (int a = 0; a < 3; ++a) v.f[a][0] = v.f[a][1] = 1.0;
            }
            v.xo = __ldg(xb + o);
            v.av = need_aux ? __ldg(ab + o) : 0.0;
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                const bool hi = (((L >> a) & 1) != 0) != (((sb >> a) & 1) != 0);   // implicit side is global +a
                v.xn[a] = need_x ? __ldg(xb + (hi ? o - Sgi[a] : o + Sgi[a])) : 0.0;
            }
        };
        // r0 and the couplings alpha c toward the implicit sides (DESIGN R-7), zeros if inactive
        auto put = [&](bool on, int e, int L, int mz, const In &v) {
            double r0 = 0.0, c[3] = {0.0, 0.0, 0.0};
            if (on) {
                const double ap = (((v.f[0][0] + v.f[0][1]) + (v.f[1][0] + v.f[1][1])) + (v.f[2][0] + v.f[2][1])) + G.beta;
                bool hi[3];
#pragma unroll
                for (int a = 0; a < 3; ++a) hi[a] = (((L >> a) & 1) != 0) != (((sb >> a) & 1) != 0);
                double al;
                if (!A.tri) {
                    const double w_ = A.omega[sb ^ L];             // the node's own box's direction bits
                    al = div_rn(w_, ap);
                    double ev = v.av;
#pragma unroll
                    for (int a = 0; a < 3; ++a) ev = fma(hi[a] ? v.f[a][0] : v.f[a][1], v.xn[a], ev);
                    r0 = fma(al, ev, (1.0 - w_) * v.xo);
                } else {
                    al = A.invd_mode ? v.av : div_rn(A.omega[0], ap);
                    r0 = A.rscale ? al * v.xo : A.coef * v.xo;
                }
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    // no coupling across an uncoupled start face: the oracle omits the term (physical
                    // boundary) and the first pass of the transposed solve must not see the neighbour box
                    const bool cut = !((L >> a) & 1) && ((mz >> a) & 1) && !((cb >> a) & 1);
                    c[a] = cut ? 0.0 : al * (hi[a] ? v.f[a][1] : v.f[a][0]);
                }
            }
            X[e] = r0;
            C0[e] = c[0];
            C1[e] = c[1];
            C2[e] = c[2];
        };
        const int warp = tid >> 5, lane = tid & 31;
        const int NR = E1 * E2, NC = (T0 + 31) >> 5, NI = NR * NC;
        // items (row, 32-wide x chunk), two per warp in flight (3 / 4 / 6: 22.5 / 20.4 / 16.7 against
        // 23.2 GLUP/s at 512^3: more loads in flight do not shorten the prologue)
        constexpr int RB = 2;
        for (int it = warp; it < NI; it += RB * (k3::NT / 32)) {
            In v[RB];
            int e_[RB], L_[RB], mz_[RB];
            bool on_[RB];
#pragma unroll
            for (int h = 0; h < RB; ++h) {
                const int item = it + h * (k3::NT / 32);
                const int row = item / NC, lx = (item % NC) * 32 + lane;
                const int l1 = row % E1, l2 = row / E1;
                const int L = (l1 < 1 ? 2 : 0) | (l2 < 1 ? 4 : 0);
                const bool live = item < NI && lx < T0;
                on_[h] = live && (L & cb) == L;
                e_[h] = live ? (lx + 1) + RS * l1 + PS * l2 : -1;
                L_[h] = L;
                mz_[h] = (lx == 0 ? 1 : 0) | (l1 == 1 ? 2 : 0) | (l2 == 1 ? 4 : 0);
                load(on_[h], O0 + lx * d[0] + (l1 - 1) * d[1] + (l2 - 1) * d[2], L, v[h]);
            }
#pragma unroll
            for (int h = 0; h < RB; ++h)
                if (e_[h] >= 0) put(on_[h], e_[h], L_[h], mz_[h], v[h]);
        }
        // the column local x = -1 of every row
        for (int row = tid; row < NR; row += k3::NT) {
            const int l1 = row % E1, l2 = row / E1;
            const int L = 1 | (l1 < 1 ? 2 : 0) | (l2 < 1 ? 4 : 0);
            const bool on = (L & cb) == L;
            const int mz = (l1 == 1 ? 2 : 0) | (l2 == 1 ? 4 : 0);
            In v;
            load(on, O0 - d[0] + (l1 - 1) * d[1] + (l2 - 1) * d[2], L, v);
            put(on, RS * l1 + PS * l2, L, mz, v);
        }
        // the padding slots (x beyond E0 in every row, rows beyond E1 in every plane): zeros
        const int rp = RS - E0, pp = PS - RS * E1;
        for (int q = tid; q < rp * E1 * E2 + pp * E2; q += k3::NT) {
            int c;
            if (q < rp * E1 * E2) { const int row = q / rp; c = (row % E1) * RS + (row / E1) * PS + E0 + q % rp; }
            else { const int r2 = q - rp * E1 * E2; c = (r2 / pp) * PS + RS * E1 + r2 % pp; }
            X[c] = 0.0;
            C0[c] = 0.0;
            C1[c] = 0.0;
            C2[c] = 0.0;
        }
    }
    // x-edge chain concurrent with the wavefront (lane wavefront, y and z start faces coupled)
    __shared__ int s_edge_done;
    const bool conc_x = (T1 * T2 <= 32) && __popc(cb) >= 2 && (cb & 6) == 6;
    if (tid == 0) s_edge_done = 0;
    // the pair data and the scratch start as zeros: idle wavefront lanes read them out of range,
    // and every value anyone reads must be finite (a zero coupling times garbage must stay zero)
    for (int e = tid; e < (int)(SCR + 80 - PVX); e += k3::NT) PVX[e] = 0.0;
    SW_TMARK(t_pro_own);
    SW_TADD(8, t_start, t_pro_own);
    __syncthreads();
    // pair data of the 2 x 2 face pairs the level loop solves (one coupled face; sets on two or
    // three faces are step 2): 1 / (1 - m_ba m_ab), m_ab, m_ba with a the member of lower global
    // index.  The y- and z-sheet pairs' own couplings toward each other are then zeroed in the
    // arrays, so that the wavefront evaluates every row with the same three-term formula.
    const bool fast_lines = T1 * T2 <= 32;
    if (fast_lines) {
        const int nx = T1 * T2, ny = T0 * T2, nz = T0 * T1;
        int fl = 0;
        for (int e = tid; e < nx + ny + nz; e += k3::NT) {
            int i, j, k, a;
            double *dst;
            if (e < nx) { i = 0; j = e % T1; k = e / T1; a = 0; dst = PVX + 3 * e; }
            else if (e < nx + ny) { const int f = e - nx; i = f % T0; k = f / T0; j = 0; a = 1; dst = PVY + 2 * (k * (T0 + 1) + i); }
            else { const int f = e - nx - ny; i = f % T0; j = f / T0; k = 0; a = 2; dst = PVZ + 2 * (j * (T0 + 1) + i); }
            const int m = (i == 0 ? (cb & 1) : 0) | (j == 0 ? (cb & 2) : 0) | (k == 0 ? (cb & 4) : 0);
            if (m != (1 << a)) continue;                          // not a pair on exactly this face
            const int w = wof(i, j, k), q = w - st[a];
            const double cw = CC(a, w), cq = CC(a, q);
            const bool qfirst = ((sb >> a) & 1) == 0;             // partner has the lower global index
            const double mab = qfirst ? cq : cw, mba = qfirst ? cw : cq;
            const double m11 = fma(mba, -mab, 1.0);
            fl |= !(fabs(m11) >= 1e-14);
            if (a == 0) {
                dst[0] = div_rn(1.0, m11);
                dst[1] = mab;
                dst[2] = mba;
            } else {        // the wavefront recomputes the pivot off its critical path
                dst[0] = mab;
                dst[1] = mba;
                CC(a, w) = 0.0;
                CC(a, q) = 0.0;
            }
        }
        if (fl) atomicOr(A.flag, 1);
        __syncthreads();
    }
    SW_TMARK(t_prologue);
    SW_TADD(1, t_start, t_prologue);
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
        // warp 2, z-edge in warp 3 (factored in parallel with the corner, substituted in order).
        // With the lane wavefront, the long x-edge chain runs concurrently with the x-sheet and the
        // wavefront, publishing its progress in s_edge_done; the other warps wait only for the
        // y- and z-edge chains (named barrier 1).
        const int warp = lt >> 5, lane = lt & 31;
        if (warp == 1) edge_chain<6>(X, WS, lane, T0, wof(1, 0, 0), st[0], st, sb, A.flag, (cb & 6) == 6,
                                     conc_x ? &s_edge_done : nullptr);
        else if (warp == 2) edge_chain<5>(X, WS, lane, T1, wof(0, 1, 0), st[1], st, sb, A.flag, (cb & 5) == 5);
        else if (warp == 3) edge_chain<3>(X, WS, lane, T2, wof(0, 0, 1), st[2], st, sb, A.flag, (cb & 3) == 3);
        else __syncthreads();
        if (!conc_x) __syncthreads();
        else if (warp != 1) {
            asm volatile("bar.sync 1, %0;" ::"r"(k3::NT - 32) : "memory");
            SW_JITTER_POINT();
        }
    }

    SW_TMARK(t_sets);
    SW_TADD(2, t_prologue, t_sets);
    // ---------------------------------------------------------------- 3. level loop (warp 0)
    if (fast_lines) {
        // (a) the x-face sheet (pairs (0, j, k) / (-1, j, k)), a 2D recurrence over d = j + k
        if (lt < 32 && (cb & 1)) {
            const int j = lt % T1, k = lt / T1;
            const bool on = lt < T1 * T2;
            const int m = 1 | (j == 0 ? (cb & 2) : 0) | (k == 0 ? (cb & 4) : 0);
            const int w = on ? wof(0, j, k) : wof(0, 0, 0), q = w - st[0];
            const bool qfirst = (sb & 1) == 0;
            const double *pd = PVX + 3 * (on ? lt : 0);
            const double piv = pd[0], mab = pd[1], mba = pd[2];
            const double cyw = CC(1, w), czw = CC(2, w), cyq = CC(1, q), czq = CC(2, q), r0w = X[w], r0q = X[q];
            for (int d = 0; d <= T1 + T2 - 2; ++d) {
                if (on && j + k == d && m == 1) {
                    const double rp = fma(czw, X[w - st[2]], fma(cyw, X[w - st[1]], r0w));
                    const double rq = fma(czq, X[q - st[2]], fma(cyq, X[q - st[1]], r0q));
                    const double ra = qfirst ? rq : rp, rb = qfirst ? rp : rq;
                    const double ub = fma(mba, ra, rb) * piv;
                    const double ua = fma(mab, ub, ra);
                    X[w] = qfirst ? ub : ua;
                    X[q] = qfirst ? ua : ub;
                }
                __syncwarp();
            }
        }
        SW_TMARK(t_xs);
        SW_TADDT(13, t_sets, t_xs, 0);
        // (b) all other nodes: lane (j, k) owns the x-line and updates node i = s - j - k at step
        //     s.  S and B arrive from lanes l-1 and l-T1 by shuffles, and so do the partner values
        //     of the y- and z-face sheets (which each lane on such a face carries in registers).
        //     One instruction stream for every kind of lane, each row the same three-term formula:
        //     a pair's coupling toward its partner was moved into the pair data (zero in the row),
        //     and a plain lane is a "pair" with its own node as partner and pair data (1, 0, 0),
        //     which leaves its node formula exact; the x-edge lane (solved in step 2) only reloads
        //     and forwards its values.  Idle lanes compute finite garbage that nobody reads.
        if (lt < 32) {
            const int lane = lt, nl = T1 * T2;
            const bool on = lane < nl;
            const int j = on ? lane % T1 : 0, k = on ? lane / T1 : 0;
            const bool yc = j == 0 && (cb & 2), zc = k == 0 && (cb & 4);
            const bool edge = on && yc && zc, ypair = on && yc && !zc, zpair = on && zc && !yc, pair = ypair || zpair;
            const int i0 = (cb & 1) ? 1 : 0;
            const int sa = ypair ? RS : (zpair ? PS : 0);                  // step toward the pair partner
            const int wl = wof(0, j, k);
            const bool qf = pair ? (((sb >> (ypair ? 1 : 2)) & 1) == 0) : true;   // partner first in index order
            const double *const pdl = ypair ? PVY + 2 * k * (T0 + 1) : (zpair ? PVZ + 2 * j * (T0 + 1) : PV1);
            const int pds = pair ? 2 : 0;
            double W = i0 ? X[wl] : 0.0;
            double Wq = (i0 && pair) ? X[wl - sa] : 0.0;                 // partner value at i0 - 1
            double u = 0.0, py = 0.0, pz = 0.0;
            const int NS = T0 + T1 + T2 - 2;
            struct Ld { double r0, cx, cy, cz, q0, qx, qy, qz, piv, mab, mba, ey, ez; };
            auto ld = [&](int s, Ld &v) {
                const int i = s - j - k;                          // any value: idle lanes read in-bounds garbage
                const int w = wl + i, q = w - sa;
                const double *pd = pdl + pds * i;
                v.r0 = X[w]; v.cx = C0[w]; v.cy = C1[w]; v.cz = C2[w];
                v.q0 = X[q]; v.qx = C0[q]; v.qy = C1[q]; v.qz = C2[q];
                v.mab = pd[0]; v.mba = pd[1];
                v.piv = div_rn(1.0, fma(v.mba, -v.mab, 1.0));    // (1 for lanes without a pair)
                v.ey = X[w - RS]; v.ez = X[w - PS];               // the x-edge lane's solved partners
            };
            auto step = [&](int s, const Ld &v) {
                const double Sv = shfl_up_f64(u, 1), Bv = shfl_up_f64(u, T1);
                const double Sq = shfl_up_f64(pz, 1), Bq = shfl_up_f64(py, T1);
                const int i = s - j - k;
                const bool act = on && i >= i0 && i < T0;
                // rows in axis order x, y, z (the pair axis has a zero coupling)
                const double rp = fma(v.cz, Bv, fma(v.cy, Sv, fma(v.cx, W, v.r0)));
                const double rq = fma(v.qz, Bq, fma(v.qy, Sq, fma(v.qx, Wq, v.q0)));
                const double ra = qf ? rq : rp, rb = qf ? rp : rq;
                const double ub = fma(v.mba, ra, rb) * v.piv;
                const double ua = fma(v.mab, ub, ra);
                double un = qf ? ub : ua;
                const double pv = qf ? ua : ub;
                un = edge ? v.r0 : un;
                st_shared_if(X + wl + i, un, act && !edge);
                u = un;
                W = sel_f64(act, un, W);              // idle (joining) lanes keep W = value at i0 - 1
                Wq = sel_f64(act, pv, Wq);
                py = ypair ? pv : v.ey;
                pz = zpair ? pv : v.ez;
            };
            // the edge lane's loads of x-edge set `need` wait until warp 1 has stored it
            auto wait_edge = [&](int need) {
                if (conc_x && need < T0) {
                    int got;
                    do {
                        asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];" : "=r"(got) : "r"(smem_u32(&s_edge_done)) : "memory");
                    } while (got < need);
                    SW_JITTER_POINT();
                }
            };
            Ld va, vb;
            __syncwarp();                             // converged (the shuffles' fast path)
            ld(0, va);
            int s = 0;
#pragma unroll 1
            for (; s + 1 < NS; s += 2) {
                wait_edge(s + 1);
                ld(s + 1, vb);
                step(s, va);
                wait_edge(s + 2);
                ld(s + 2, va);
                step(s + 1, vb);
            }
            if (s < NS) step(s, va);
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
    SW_TADD(3, t_sets, t_levels);

    // ---------------------------------------------------------------- 4. write-back of the box
    // row-wise like the prologue: a warp per (local y, z) row, lanes along x (one coalesced run)
    {
        const int warp = tid >> 5, lane = tid & 31;
        const int NC = (T0 + 31) >> 5, NI = T1 * T2 * NC;
        const int64_t d1 = ((sb >> 1) & 1) ? -P0 : P0, d2 = ((sb >> 2) & 1) ? -P01 : P01;
        const int d0 = (sb & 1) ? -1 : 1;
        double *const ob = A.out + gbase + (2 + ((sb & 1) ? T0 - 1 : 0)) + (2 + (((sb >> 1) & 1) ? T1 - 1 : 0)) * P0 +
                           (2 + (((sb >> 2) & 1) ? T2 - 1 : 0)) * P01;
        for (int item = warp; item < NI; item += k3::NT / 32) {
            const int row = item / NC, lx = (item % NC) * 32 + lane;
            const int l1 = row % T1, l2 = row / T1;
            if (lx < T0) ob[lx * d0 + l1 * d1 + l2 * d2] = X[wof(lx, l1, l2)];
        }
    }
    SW_TMARK(t_end);
    SW_TADD(4, t_levels, t_end);
    SW_TADD(5, 0, 1);
}

// Strides of the compact arrays: the smallest padded (RS, PS) for which the 64-bit accesses of the
// wavefront's lanes (j, k) = (l % T1, l / T1), l < T1 T2, are free of bank conflicts within each
// half-warp (or have the fewest conflicts).
inline void sweep3_layout(const int T[3], int *RS, int *PS) {
    if (T[0] == 32 && T[1] == 8 && T[2] == 4) { *RS = 34; *PS = 307; return; }   // Shape3<1>
    const int E0 = T[0] + 1, E1 = T[1] + 1, nl = T[1] * T[2];
    int best = 1 << 30;
    for (int rs = E0; rs < E0 + 16; ++rs)
        for (int ps = rs * E1; ps < rs * E1 + 16; ++ps) {
            int worst = 0;
            for (int h = 0; h < 2; ++h) {
                int cnt[16] = {0};
                for (int l = 16 * h; l < 16 * h + 16 && l < nl; ++l) {
                    const int off = rs * (l % T[1]) + ps * (l / T[1]);
                    const int c = ++cnt[off & 15];
                    if (c > worst) worst = c;
                }
            }
            const int score = worst * (1 << 20) + ps;       // fewest conflicts, then least memory
            if (score < best) { best = score; *RS = rs; *PS = ps; }
        }
}

inline size_t sweep3_smem(const Geo &G) {
    int rs, ps;
    sweep3_layout(G.T, &rs, &ps);
    const size_t ws = (size_t)ps * (G.T[2] + 1);
    const size_t pv = 3 * (size_t)G.T[1] * G.T[2] + 2 * (size_t)(G.T[0] + 1) * (G.T[1] + G.T[2]) + 4;
    return sizeof(double) * (4 * ws + pv + 80);
}

// the fast 3D path handles boxes whose compact arrays fit in shared memory
inline bool sweep3_supported(const Geo &G) {
    if (G.dim != 3) return false;
    return (G.T[0] % 2 == 0) && sweep3_smem(G) <= 227 * 1024 && G.T[1] * G.T[2] <= k3::MAXLINES &&
           G.T[0] <= 33 && G.T[1] <= 33 && G.T[2] <= 33 && G.off[0] == 0 && G.off[1] == 0;
}

template <bool FACES, int SHAPE>
inline void launch_sweep3_t(const Sweep3Args &A, size_t smem, unsigned tiles, cudaStream_t s) {
    cudaFuncSetAttribute(k_sweep3<FACES, SHAPE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_sweep3<FACES, SHAPE><<<tiles, k3::NT, smem, s>>>(A);
}

inline cudaError_t launch_sweep3(const Sweep3Args &A0, cudaStream_t s) {
    Sweep3Args A = A0;
    sweep3_layout(A.G.T, &A.RS, &A.PS);
    const size_t smem = sweep3_smem(A.G);
    const bool faces = A.f0 != nullptr;
    const bool c5 = A.G.T[0] == 32 && A.G.T[1] == 8 && A.G.T[2] == 4;
    const unsigned tiles = (unsigned)((int64_t)A.G.nt[0] * A.G.nt[1] * A.G.nt[2]);
    if (faces) {
        if (c5) launch_sweep3_t<true, 1>(A, smem, tiles, s);
        else launch_sweep3_t<true, 0>(A, smem, tiles, s);
    } else {
        if (c5) launch_sweep3_t<false, 1>(A, smem, tiles, s);
        else launch_sweep3_t<false, 0>(A, smem, tiles, s);
    }
    return cudaGetLastError();
}

}  // namespace sw
