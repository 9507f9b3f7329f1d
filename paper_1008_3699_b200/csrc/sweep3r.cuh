// sweep3r.cuh -- 3D decomposed sweep / block-triangular solve, rolling warp-specialised version for
// boxes with T1 * T2 <= 32 lines and T0 <= 32 (config 5's 32 x 8 x 4), sm_100a.
//
// Same arithmetic as k_sweep3 (sweep3.cuh), so the result is bitwise that of the oracle; what changes
// is how a CTA spends its time.  In k_sweep3 one warp runs a box's 42-step wavefront while the other
// three wait at a barrier, and the next box cannot start before the whole box is written back: the
// SM is latency bound at ~0.35 issue utilisation (profiles/r02f_*).  Here each CTA is persistent and
// walks a list of boxes with ONE set of compact arrays (X, C0..C2 over the extended box, as in
// k_sweep3) that is refilled column by column behind the running wavefront:
//   warp 0     the lane wavefront of box q (lane (j, k) owns the x-line, node s - j - k at step s),
//              storing each result straight to global memory;
//   warp 1     the x-edge chain of box q (4 x 4 sets along x, factored per chunk, substituted in
//              order), published to the wavefront step by step;
//   warp 2     box q's corner set, y- and z-edge chains, x-face sheet (and its write-back), and the
//              y/z-sheet pair data per chunk of columns;
//   warps 3-4  producers: r0 and the couplings of box q+1, chunk by chunk of compact x-columns
//              [0,2), [2,10), [10,18), [18,26), [26,33), each chunk as soon as box q's wavefront has read its
//              columns for the last time (lane j + k = D reads column c last at step c - 1 + D).
// Progress is exchanged through monotone counters in shared memory (st.release / ld.acquire; a box
// q adds q * BASE), so every wait is a spin on a flag of the same CTA.  The x = 0 column of a box
// whose x start face is coupled is solved by the sheet (warp 2) and written back there; all other
// nodes are written by the wavefront lane that computes them.
#pragma once
#include "sweep3.cuh"

namespace sw {

namespace k3r {
constexpr int NW = 5;               // warps per CTA
constexpr int NT = NW * 32;
constexpr int PW0 = 3;              // first producer warp
constexpr int NPT = (NW - PW0) * 32;   // producer threads
constexpr int BASE = 256;           // per-box stride of the progress counters (> steps, chunks)
constexpr int CW = 8;               // chunk width in compact columns (chunk 0 has one more: local x = -1)
}  // namespace k3r

__device__ __forceinline__ int ld_acq(const int *p) {
    int v;
    asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
    return v;
}
__device__ __forceinline__ void st_rel(int *p, int v) {
    asm volatile("st.release.cta.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
// Progress of the wavefront (a write-after-read hand-off: the producers may overwrite columns the
// wavefront has finished reading).  A release store here would compile to MEMBAR.ALL.CTA, which
// waits for the wavefront's outstanding global stores of the results; the reads it must order
// are shared loads whose values were consumed by the steps that preceded the store (register
// dependences: every load of a released column fed a shuffle or FMA of an earlier, completed
// step), so a relaxed store suffices.
__device__ __forceinline__ void st_progress(int *p, int v) {
    asm volatile("st.relaxed.cta.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
// every lane of the calling warp spins until *p >= v (a broadcast shared load); with SW_TRACE the
// cycles waited are added to *acc
__device__ __forceinline__ void wait_ge(const int *p, int v, long long *acc = nullptr) {
    if (ld_acq(p) < v) {
#ifdef SW_TRACE
        const long long t0 = sw_clock();
#endif
        unsigned ns = 32;
        do {
            __nanosleep(ns);
            ns = ns < 512 ? 2 * ns : 512;
        } while (ld_acq(p) < v);
#ifdef SW_TRACE
        if (acc) *acc += sw_clock() - t0;
#endif
    }
    SW_JITTER_POINT();
}
#ifdef SW_TRACE
#define SW_T3(var) const long long var = sw_clock()
#define SW_T3ADD(slot, a) tr[slot] += sw_clock() - (a)
#else
#define SW_T3(var)
#define SW_T3ADD(slot, a)
#endif

// first compact column of chunk k: chunk 0 = compact [0, 2) (local x = -1, 0: everything the corner,
// the y / z edges and the x-sheet need, so they can start early), then CW columns per chunk
__device__ __forceinline__ int chunk_start(int k, int E0) {
    const int c = k == 0 ? 0 : 2 + k3r::CW * (k - 1);
    return c < E0 ? c : E0;
}
__device__ __forceinline__ int chunk_count(int E0) { return 1 + (E0 - 2 + k3r::CW - 1) / k3r::CW; }

struct Box3i {
    int sb, cb;
    int64_t gbase;   // padded index of box min - (2, 2, 2)
};

template <int SHAPE>
__device__ __forceinline__ Box3i box3_info(const Sweep3Args &A, int64_t b) {
    using SH = Shape3<SHAPE>;
    const Geo &G = A.G;
    const int T0 = SH::t0(A), T1 = SH::t1(A), T2 = SH::t2(A);
    const int tx = (int)(b % G.nt[0]);
    const int ty = (int)((b / G.nt[0]) % G.nt[1]);
    const int tz = (int)(b / ((int64_t)G.nt[0] * G.nt[1]));
    const int64_t R[3] = {tx, ty, tz + G.toff[2]};
    Box3i B;
    B.sb = 0;
    B.cb = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const int s = ((A.base >> a) & 1) ^ (int)(R[a] & 1);
        const bool c = A.couple && (s ? (R[a] < G.ntg[a] - 1) : (R[a] > 0));
        B.sb |= s << a;
        B.cb |= (int)c << a;
    }
    B.gbase = (int64_t)tz * T2 * G.P01 + (int64_t)ty * T1 * G.P0 + (int64_t)tx * T0;
    return B;
}

// one edge chain inside one warp: lane t-1 factors set t, then the sets are substituted in order
template <int AXES>
__device__ __forceinline__ void edge_chain_w(double *X, int WS, int lane, int T, int w1, int step, const int st[3],
                                             int sbits, int *flag) {
    Fac4 F;
    int fl = 0;
    const bool mine = lane + 1 < T;
    if (mine) factor4<AXES>(X, WS, w1 + lane * step, st, sbits, F, fl);
    if (fl) atomicOr(flag, 1);
    __syncwarp();
    for (int t = 1; t < T; ++t) {
        if (lane == t - 1) subst4<AXES>(X, WS, w1 + (t - 1) * step, st, sbits, F);
        __syncwarp();
    }
}

template <bool FACES, int SHAPE>
__global__ void __launch_bounds__(k3r::NT, 4) k_sweep3r(Sweep3Args A, int64_t nbox) {
    extern __shared__ __align__(128) double sm[];
    __shared__ int s_wf, s_prod, s_pd, s_set, s_xe;
    SW_JITTER_POINT();
    const Geo &G = A.G;
    using SH = Shape3<SHAPE>;
    const int T0 = SH::t0(A), T1 = SH::t1(A), T2 = SH::t2(A);
    const int E0 = T0 + 1, E1 = T1 + 1, E2 = T2 + 1;
    const int RS = SH::rs(A), PS = SH::ps(A);
    const int WS = PS * E2;
    double *const X = sm;
    double *const C0 = sm + WS, *const C1 = sm + 2 * WS, *const C2 = sm + 3 * WS;
    double *const PVX = sm + 4 * WS;
    double *const PVY = PVX + 3 * T1 * T2;
    double *const PVZ = PVY + 2 * (T0 + 1) * T2;
    double *const PV1 = PVZ + 2 * (T0 + 1) * T1;
    double *const SCR = PV1 + 4;
    auto CC = [&](int a, int w) -> double & { return sm[(a + 1) * WS + w]; };
    auto wof = [&](int l0, int l1, int l2) { return (l0 + 1) + RS * (l1 + 1) + PS * (l2 + 1); };
    const int st[3] = {1, RS, PS};
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int NS = T0 + T1 + T2 - 2;        // wavefront steps
    const int D = T1 + T2 - 2;              // largest j + k of a line
    const int nch = chunk_count(E0);
    const int64_t P0 = G.P0, P01 = G.P01;
    // boxes of this CTA: b = blockIdx.x + q gridDim.x
    const int nq = (int)((nbox - blockIdx.x + gridDim.x - 1) / gridDim.x);

    // ---------------------------------------------------------------- set-up
    // every slot starts finite (idle lanes read out of their lines; zero couplings times garbage must
    // stay zero), the padding slots of the compact arrays stay zero for good
    for (int e = tid; e < 4 * WS + (int)(SCR + 80 - PVX); e += k3r::NT) sm[e] = 0.0;
    if (tid == 0) {
        s_wf = 0;
        s_prod = 0;
        s_pd = 0;
        s_set = 0;
        s_xe = 0;
    }
    __syncthreads();
    long long tr[16] = {0};                 // SW_TRACE: per-role wait / busy cycles (lane 0 of each role)
    SW_T3(t_begin);

    if (warp >= k3r::PW0) {
        // ============================================================ producers
        const int pt = tid - k3r::PW0 * 32;
        const int P0i = (int)P0, P01i = (int)P01;
        const int Sgi[3] = {1, P0i, P01i};
        const bool need_x = !A.tri, need_aux = !A.tri || A.invd_mode;
        for (int q = 0; q < nq; ++q) {
            const Box3i bx = box3_info<SHAPE>(A, blockIdx.x + (int64_t)q * gridDim.x);
            const int sb = bx.sb, cb = bx.cb;
            int O0 = 0, d[3];
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                const int Ta = a == 0 ? T0 : (a == 1 ? T1 : T2);
                const bool sa_ = (sb >> a) & 1;
                O0 += (2 + (sa_ ? Ta - 1 : 0)) * Sgi[a];
                d[a] = sa_ ? -Sgi[a] : Sgi[a];
            }
            const double *__restrict__ xb = A.xin + bx.gbase;
            const double *__restrict__ ab = (A.aux ? A.aux : A.xin) + bx.gbase;
            const double *__restrict__ f0b = (FACES ? A.f0 : A.xin) + bx.gbase;
            const double *__restrict__ f1b = (FACES ? A.f1 : A.xin) + bx.gbase;
            const double *__restrict__ f2b = (FACES ? A.f2 : A.xin) + bx.gbase;
            for (int k = 0; k < nch; ++k) {
                const int c0 = chunk_start(k, E0), c1 = chunk_start(k + 1, E0), ncol = c1 - c0;
                // box q-1's wavefront has read columns < c1 for the last time
                if (q > 0) wait_ge(&s_wf, (q - 1) * k3r::BASE + min(c1 + D, NS), &tr[0]);
                const int n = E1 * E2 * ncol;
                constexpr int KB = 2;
                for (int n0 = pt; n0 < n; n0 += KB * k3r::NPT) {
                    double f[KB][3][2], xn[KB][3], xo[KB], av[KB];
                    int e_[KB], L_[KB], mz_[KB];
                    bool on_[KB];
#pragma unroll
                    for (int h = 0; h < KB; ++h) {
                        const int nn = n0 + h * k3r::NPT;
                        const int row = nn / ncol, cc = c0 + nn % ncol;     // compact column
                        const int l1 = row % E1, l2 = row / E1, lx = cc - 1;
                        const int L = (lx < 0 ? 1 : 0) | (l1 < 1 ? 2 : 0) | (l2 < 1 ? 4 : 0);
                        const bool live = nn < n;
                        on_[h] = live && (L & cb) == L;
                        e_[h] = live ? cc + RS * l1 + PS * l2 : -1;
                        L_[h] = L;
                        mz_[h] = (lx == 0 ? 1 : 0) | (l1 == 1 ? 2 : 0) | (l2 == 1 ? 4 : 0);
                        if (on_[h]) {
                            const int o = O0 + lx * d[0] + (l1 - 1) * d[1] + (l2 - 1) * d[2];
                            if (FACES) {
                                f[h][0][0] = __ldg(f0b + o); f[h][0][1] = __ldg(f0b + o + 1);
                                f[h][1][0] = __ldg(f1b + o); f[h][1][1] = __ldg(f1b + o + P0i);
                                f[h][2][0] = __ldg(f2b + o); f[h][2][1] = __ldg(f2b + o + P01i);
                            } else {
#pragma unroll
                                for (int a = 0; a < 3; ++a) f[h][a][0] = f[h][a][1] = 1.0;
                            }
                            xo[h] = __ldg(xb + o);
                            av[h] = need_aux ? __ldg(ab + o) : 0.0;
#pragma unroll
                            for (int a = 0; a < 3; ++a) {
                                const bool hi = (((L >> a) & 1) != 0) != (((sb >> a) & 1) != 0);
                                xn[h][a] = need_x ? __ldg(xb + (hi ? o - Sgi[a] : o + Sgi[a])) : 0.0;
                            }
                        }
                    }
#pragma unroll
                    for (int h = 0; h < KB; ++h) {
                        const int e = e_[h];
                        if (e < 0) continue;
                        const int L = L_[h];
                        double r0 = 0.0, c[3] = {0.0, 0.0, 0.0};
                        if (on_[h]) {
                            const double(&fk)[3][2] = f[h];
                            const double ap =
                                (((fk[0][0] + fk[0][1]) + (fk[1][0] + fk[1][1])) + (fk[2][0] + fk[2][1])) + G.beta;
                            bool hi[3];
#pragma unroll
                            for (int a = 0; a < 3; ++a) hi[a] = (((L >> a) & 1) != 0) != (((sb >> a) & 1) != 0);
                            double al;
                            if (!A.tri) {
                                const double w_ = A.omega[sb ^ L];
                                al = div_rn(w_, ap);
                                double ev = av[h];
#pragma unroll
                                for (int a = 0; a < 3; ++a) ev = fma(hi[a] ? fk[a][0] : fk[a][1], xn[h][a], ev);
                                r0 = fma(al, ev, (1.0 - w_) * xo[h]);
                            } else {
                                al = A.invd_mode ? av[h] : div_rn(A.omega[0], ap);
                                r0 = A.rscale ? al * xo[h] : A.coef * xo[h];
                            }
#pragma unroll
                            for (int a = 0; a < 3; ++a) {
                                const bool cut = !((L >> a) & 1) && ((mz_[h] >> a) & 1) && !((cb >> a) & 1);
                                c[a] = cut ? 0.0 : al * (hi[a] ? fk[a][1] : fk[a][0]);
                            }
                        }
                        X[e] = r0;
                        C0[e] = c[0];
                        C1[e] = c[1];
                        C2[e] = c[2];
                    }
                }
                asm volatile("bar.sync 2, %0;" ::"r"(k3r::NPT) : "memory");   // the producers' chunk is in place
                SW_JITTER_POINT();
                if (pt == 0) st_rel(&s_prod, q * k3r::BASE + k + 1);
            }
        }
    } else if (warp == 2) {
        // ============================================================ sets, x-sheet, pair data
        for (int q = 0; q < nq; ++q) {
            const Box3i bx = box3_info<SHAPE>(A, blockIdx.x + (int64_t)q * gridDim.x);
            const int sb = bx.sb, cb = bx.cb;
            const int qb = q * k3r::BASE;
            // pair data of the y- and z-sheet pairs (exactly one coupled face) of local x in [x0, x1),
            // their couplings toward each other zeroed in the arrays (k_sweep3's "pair data" step)
            auto pair_data = [&](int x0, int x1) {
                int fl = 0;
                const int ny = (x1 - x0) * T2, nz = (x1 - x0) * T1;
                for (int e = lane; e < ny + nz; e += 32) {
                    int i, j, k, a;
                    double *dst;
                    if (e < ny) { i = x0 + e % (x1 - x0); k = e / (x1 - x0); j = 0; a = 1; dst = PVY + 2 * (k * (T0 + 1) + i); }
                    else { const int f = e - ny; i = x0 + f % (x1 - x0); j = f / (x1 - x0); k = 0; a = 2; dst = PVZ + 2 * (j * (T0 + 1) + i); }
                    const int m = (i == 0 ? (cb & 1) : 0) | (j == 0 ? (cb & 2) : 0) | (k == 0 ? (cb & 4) : 0);
                    if (m != (1 << a)) continue;
                    const int w = wof(i, j, k), qq = w - st[a];
                    const double cw = CC(a, w), cq = CC(a, qq);
                    const bool qfirst = ((sb >> a) & 1) == 0;
                    const double mab = qfirst ? cq : cw, mba = qfirst ? cw : cq;
                    const double m11 = fma(mba, -mab, 1.0);
                    fl |= !(fabs(m11) >= 1e-14);
                    dst[0] = mab;
                    dst[1] = mba;
                    CC(a, w) = 0.0;
                    CC(a, qq) = 0.0;
                }
                if (fl) atomicOr(A.flag, 1);
            };
            wait_ge(&s_prod, qb + 1, &tr[2]);                           // chunk 0 of box q
            __syncwarp();
            SW_T3(t_sets0);
            // x-sheet pair data (x = 0 column): 1 / pivot, m_ab, m_ba
            if (cb & 1) {
                int fl = 0;
                for (int e = lane; e < T1 * T2; e += 32) {
                    const int j = e % T1, k = e / T1;
                    const int m = 1 | (j == 0 ? (cb & 2) : 0) | (k == 0 ? (cb & 4) : 0);
                    if (m != 1) continue;
                    const int w = wof(0, j, k), qq = w - st[0];
                    const double cw = CC(0, w), cq = CC(0, qq);
                    const bool qfirst = (sb & 1) == 0;
                    const double mab = qfirst ? cq : cw, mba = qfirst ? cw : cq;
                    const double m11 = fma(mba, -mab, 1.0);
                    fl |= !(fabs(m11) >= 1e-14);
                    PVX[3 * e] = div_rn(1.0, m11);
                    PVX[3 * e + 1] = mab;
                    PVX[3 * e + 2] = mba;
                }
                if (fl) atomicOr(A.flag, 1);
            }
            pair_data(0, min(chunk_start(1, E0) - 1, T0));
            __syncwarp();
            // corner set and the y- / z-edge chains (sets on two or three coupled faces)
            if (__popc(cb) >= 2) {
                if (cb == 7) {
                    corner8_coop(X, WS, SCR, lane, wof(0, 0, 0), st, sb, A.flag);
                } else if (lane == 0) {
                    const int w = wof(0, 0, 0);
                    switch (cb) {
                        case 3: solve_set3<3>(X, WS, w, st, sb, A.flag); break;
                        case 5: solve_set3<5>(X, WS, w, st, sb, A.flag); break;
                        default: solve_set3<6>(X, WS, w, st, sb, A.flag); break;
                    }
                }
                __syncwarp();
                if ((cb & 5) == 5) edge_chain_w<5>(X, WS, lane, T1, wof(0, 1, 0), st[1], st, sb, A.flag);
                if ((cb & 3) == 3) edge_chain_w<3>(X, WS, lane, T2, wof(0, 0, 1), st[2], st, sb, A.flag);
            }
            SW_T3ADD(4, t_sets0);
            SW_T3(t_sheet0);
            // the x-face sheet (pairs (0, j, k) / (-1, j, k)), a 2D recurrence over d = j + k, and the
            // write-back of the box's x = 0 column (the wavefront starts at x = 1)
            if (cb & 1) {
                const int j = lane % T1, k = lane / T1;
                const bool on = lane < T1 * T2;
                const int m = 1 | (j == 0 ? (cb & 2) : 0) | (k == 0 ? (cb & 4) : 0);
                const int w = on ? wof(0, j, k) : wof(0, 0, 0), qq = w - st[0];
                const bool qfirst = (sb & 1) == 0;
                const double *pd = PVX + 3 * (on ? lane : 0);
                const double piv = pd[0], mab = pd[1], mba = pd[2];
                const double cyw = CC(1, w), czw = CC(2, w), cyq = CC(1, qq), czq = CC(2, qq), r0w = X[w], r0q = X[qq];
                for (int dd = 0; dd <= T1 + T2 - 2; ++dd) {
                    if (on && j + k == dd && m == 1) {
                        const double rp = fma(czw, X[w - st[2]], fma(cyw, X[w - st[1]], r0w));
                        const double rq = fma(czq, X[qq - st[2]], fma(cyq, X[qq - st[1]], r0q));
                        const double ra = qfirst ? rq : rp, rb = qfirst ? rp : rq;
                        const double ub = fma(mba, ra, rb) * piv;
                        const double ua = fma(mab, ub, ra);
                        X[w] = qfirst ? ub : ua;
                        X[qq] = qfirst ? ua : ub;
                    }
                    __syncwarp();
                }
                __syncwarp();
            }
            SW_T3ADD(5, t_sheet0);
            // the x = 0 column's values: read before the release (they stay in place until the
            // wavefront of box q is past column 1), stored to global after it (a release would
            // otherwise wait for these global stores)
            double x0v = 0.0;
            const bool wr0 = (cb & 1) && lane < T1 * T2;
            if (wr0) x0v = X[wof(0, lane % T1, lane / T1)];
            __syncwarp();
            if (lane == 0) {
                st_rel(&s_pd, qb + 1);
                st_rel(&s_set, q + 1);
            }
            if (wr0) {
                const int64_t d1 = ((sb >> 1) & 1) ? -P0 : P0, d2 = ((sb >> 2) & 1) ? -P01 : P01;
                double *const ob = A.out + bx.gbase + (2 + ((sb & 1) ? T0 - 1 : 0)) +
                                   (2 + (((sb >> 1) & 1) ? T1 - 1 : 0)) * P0 + (2 + (((sb >> 2) & 1) ? T2 - 1 : 0)) * P01;
                ob[(lane % T1) * d1 + (lane / T1) * d2] = x0v;
            }
            // the other chunks' pair data, as the producers deliver them
            for (int k = 1; k < nch; ++k) {
                wait_ge(&s_prod, qb + k + 1, &tr[3]);
                __syncwarp();
                pair_data(chunk_start(k, E0) - 1, chunk_start(k + 1, E0) - 1);
                __syncwarp();
                if (lane == 0) st_rel(&s_pd, qb + k + 1);
            }
        }
    } else if (warp == 1) {
        // ============================================================ x-edge chain
        for (int q = 0; q < nq; ++q) {
            const Box3i bx = box3_info<SHAPE>(A, blockIdx.x + (int64_t)q * gridDim.x);
            const int sb = bx.sb, cb = bx.cb;
            const int qb = q * k3r::BASE;
            if ((cb & 6) != 6) continue;
            wait_ge(&s_set, q + 1, &tr[6]);         // the corner set (set 0) is in place
            for (int k = 0; k < nch; ++k) {
                wait_ge(&s_prod, qb + k + 1, &tr[7]);
                __syncwarp();
                const int t0 = max(chunk_start(k, E0) - 1, 1), t1 = min(chunk_start(k + 1, E0) - 1, T0);
                Fac4 F;
                int fl = 0;
                const int t = t0 + lane;
                if (t < t1) factor4<6>(X, WS, wof(t, 0, 0), st, sb, F, fl);
                if (fl) atomicOr(A.flag, 1);
                __syncwarp();
                for (int u = t0; u < t1; ++u) {
                    if (lane == u - t0) {
                        subst4<6>(X, WS, wof(u, 0, 0), st, sb, F);
                        st_rel(&s_xe, qb + u);          // set u is in place
                    }
                    __syncwarp();
                }
            }
            if (lane == 0) st_rel(&s_xe, qb + T0);
        }
    } else {
        // ============================================================ warp 0: the wavefront
        for (int q = 0; q < nq; ++q) {
            const Box3i bx = box3_info<SHAPE>(A, blockIdx.x + (int64_t)q * gridDim.x);
            const int sb = bx.sb, cb = bx.cb;
            const int qb = q * k3r::BASE;
            const bool conc_x = (cb & 6) == 6;
            wait_ge(&s_set, q + 1, &tr[9]);
            __syncwarp();
            const int nl = T1 * T2;
            const bool on = lane < nl;
            const int j = on ? lane % T1 : 0, k = on ? lane / T1 : 0;
            const bool yc = j == 0 && (cb & 2), zc = k == 0 && (cb & 4);
            const bool edge = on && yc && zc, ypair = on && yc && !zc, zpair = on && zc && !yc, pair = ypair || zpair;
            const int i0 = (cb & 1) ? 1 : 0;
            const int sa = ypair ? RS : (zpair ? PS : 0);
            const int wl = wof(0, j, k);
            const bool qf = pair ? (((sb >> (ypair ? 1 : 2)) & 1) == 0) : true;
            const double *const pdl = ypair ? PVY + 2 * k * (T0 + 1) : (zpair ? PVZ + 2 * j * (T0 + 1) : PV1);
            const int pds = pair ? 2 : 0;
            // global address of local (0, j, k) and the step of local +x
            const int64_t d1 = ((sb >> 1) & 1) ? -P0 : P0, d2 = ((sb >> 2) & 1) ? -P01 : P01;
            const int d0 = (sb & 1) ? -1 : 1;
            double *const orow = A.out + bx.gbase + (2 + ((sb & 1) ? T0 - 1 : 0)) +
                                 (2 + (((sb >> 1) & 1) ? T1 - 1 : 0)) * P0 + (2 + (((sb >> 2) & 1) ? T2 - 1 : 0)) * P01 +
                                 j * d1 + k * d2;
            double W = i0 ? X[wl] : 0.0;
            double Wq = (i0 && pair) ? X[wl - sa] : 0.0;
            double u = 0.0, py = 0.0, pz = 0.0;
            struct Ld { double r0, cx, cy, cz, q0, qx, qy, qz, piv, mab, mba, ey, ez; };
            int ready = chunk_start(1, E0);          // compact columns < ready have their pair data
            auto ld = [&](int s, Ld &v) {
                // column s + 1 (lane (0, 0)'s node) and everything below must be delivered
                if (s + 1 >= ready && ready < E0) {
                    int kk = 1;
                    while (chunk_start(kk + 1, E0) <= s + 1 && kk + 1 < nch) ++kk;
                    wait_ge(&s_pd, qb + kk + 1, &tr[10]);
                    ready = chunk_start(kk + 1, E0);
                }
                const int i = s - j - k;
                const int w = wl + i, qq = w - sa;
                const double *pd = pdl + pds * i;
                v.r0 = X[w]; v.cx = C0[w]; v.cy = C1[w]; v.cz = C2[w];
                v.q0 = X[qq]; v.qx = C0[qq]; v.qy = C1[qq]; v.qz = C2[qq];
                v.mab = pd[0]; v.mba = pd[1];
                v.piv = div_rn(1.0, fma(v.mba, -v.mab, 1.0));
                v.ey = X[w - RS]; v.ez = X[w - PS];
            };
            auto step = [&](int s, const Ld &v) {
                const double Sv = shfl_up_f64(u, 1), Bv = shfl_up_f64(u, T1);
                const double Sq = shfl_up_f64(pz, 1), Bq = shfl_up_f64(py, T1);
                const int i = s - j - k;
                const bool act = on && i >= i0 && i < T0;
                const double rp = fma(v.cz, Bv, fma(v.cy, Sv, fma(v.cx, W, v.r0)));
                const double rq = fma(v.qz, Bq, fma(v.qy, Sq, fma(v.qx, Wq, v.q0)));
                const double ra = qf ? rq : rp, rb = qf ? rp : rq;
                const double ub = fma(v.mba, ra, rb) * v.piv;
                const double ua = fma(v.mab, ub, ra);
                double un = qf ? ub : ua;
                const double pv = qf ? ua : ub;
                un = edge ? v.r0 : un;              // (the x-edge lane's node: solved by the chain)
                if (act) orow[(int64_t)i * d0] = un;
                u = un;
                W = sel_f64(act, un, W);
                Wq = sel_f64(act, pv, Wq);
                py = ypair ? pv : v.ey;
                pz = zpair ? pv : v.ez;
            };
            auto wait_edge = [&](int need) {
                if (conc_x && need < T0) wait_ge(&s_xe, qb + need, &tr[11]);
            };
            Ld va, vb;
            __syncwarp();
            ld(0, va);                              // (set 0, the corner, is in place: s_set)
            int s = 0;
#pragma unroll 1
            for (; s + 1 < NS; s += 2) {
                wait_edge(s + 1);
                ld(s + 1, vb);
                step(s, va);
                wait_edge(s + 2);
                ld(s + 2, va);
                step(s + 1, vb);
                __syncwarp();
                if (lane == 0) st_progress(&s_wf, qb + s + 2);
            }
            if (s < NS) step(s, va);
            __syncwarp();
            if (lane == 0) st_progress(&s_wf, qb + NS);
        }
    }
#ifdef SW_TRACE
    // roles: 0 producer wait, 1 producer total, 2/3 warp 2 waits, 4 sets, 5 sheet, 6/7 warp 1 waits,
    // 9/10/11 wavefront waits, 12 wavefront total, 13 warp 2 total, 14 warp 1 total, 15 boxes
    const long long tot = sw_clock() - t_begin;
    if (lane == 0 && (warp <= 2 || tid == k3r::PW0 * 32)) {
        const int role_tot = warp == 0 ? 12 : (warp == 1 ? 14 : (warp == 2 ? 13 : 1));
        tr[role_tot] = tot;
        if (warp == 0) tr[15] = nq;
        for (int i = 0; i < 16; ++i)
            if (tr[i]) atomicAdd(&sw_trace_sum[i], (unsigned long long)tr[i]);
    }
#endif
}

inline bool sweep3r_supported(const Geo &G) {
    return sweep3_supported(G) && G.T[1] * G.T[2] <= 32 && G.T[0] <= 32;
}

template <bool FACES, int SHAPE>
inline void launch_sweep3r_t(const Sweep3Args &A, size_t smem, int64_t nbox, cudaStream_t s) {
    static int sms = 0;
    static size_t last_smem = 0, attr_smem = 0;
    static int per = 1;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    if (smem > attr_smem) {
        cudaFuncSetAttribute(k_sweep3r<FACES, SHAPE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr_smem = smem;
    }
    if (smem != last_smem) {        // persistent grid: every resident CTA slot of the device
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_sweep3r<FACES, SHAPE>, k3r::NT, smem);
        if (per < 1) per = 1;
        last_smem = smem;
    }
    const int64_t ctas = (int64_t)sms * per;
    const int64_t grid = nbox < ctas ? nbox : ctas;
    k_sweep3r<FACES, SHAPE><<<(unsigned)grid, k3r::NT, smem, s>>>(A, nbox);
}

inline cudaError_t launch_sweep3r(const Sweep3Args &A0, cudaStream_t s) {
    Sweep3Args A = A0;
    sweep3_layout(A.G.T, &A.RS, &A.PS);
    const size_t smem = sweep3_smem(A.G);
    const bool faces = A.f0 != nullptr;
    const bool c5 = A.G.T[0] == 32 && A.G.T[1] == 8 && A.G.T[2] == 4;
    const int64_t nbox = (int64_t)A.G.nt[0] * A.G.nt[1] * A.G.nt[2];
    if (faces) {
        if (c5) launch_sweep3r_t<true, 1>(A, smem, nbox, s);
        else launch_sweep3r_t<true, 0>(A, smem, nbox, s);
    } else {
        if (c5) launch_sweep3r_t<false, 1>(A, smem, nbox, s);
        else launch_sweep3r_t<false, 0>(A, smem, nbox, s);
    }
    return cudaGetLastError();
}

}  // namespace sw
