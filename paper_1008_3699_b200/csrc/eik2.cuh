// eik2.cuh -- decomposed fast-sweeping pass for the eikonal equation |grad u| = f on the
// multi-frontal schedule, 2D (PAPER:2593-2599 names the application).  The local
// update is the Godunov rule of fast sweeping (DESIGN R-E1), neighbours' new values on the start
// side of a node's box and old values elsewhere (R-E2), the coupled sets at start-start faces (the
// SOR sweep's 2-member pairs and 4-member corner) solved exactly by ordered fixing (R-E3): the same
// operations in the same order as the oracle's or_eik_sweep, so the result is bitwise equal.
//
// One CTA of 256 threads per box (T0, T1 <= 64).  All threads stage in the old values of the box and
// its 2-node halo in LOCAL coordinates (local +a points away from the box's start corner; a node
// outside the domain reads +inf) and the slowness of the active nodes (own and partner layers).
// Then the corner set (four lanes of warp 0, ordered fixing with shuffles), the two start-face chains
// (lanes 0 and 1: row 0 with its partner row, column 0 with its partner column: pairs by ordered
// fixing, or plain updates along an uncoupled face; branch-free, window operands loaded a step
// ahead), then the other own nodes front by front (d = x + y; the first 64 threads, one column
// each, a named barrier of the 64 per front): a node outside the coupled sets is updated in place
// from the window, which holds new values on its start side and old values on its end side,
// exactly the split the method prescribes.  Write-back by all threads.
// (A register wavefront in one warp -- lane l owning rows 2l+1 and 2l+2, the second a column behind
// the first -- was built and is bitwise correct, but has as many steps as there are fronts (126)
// and pays the square root on every node: 0.87 instead of 0.70 ms per pass at 4096^2; not kept,
// profiles/r02_eik_wavefront_experiment.txt.)
#pragma once
#include "common.cuh"
#include "sweep2p.cuh"

namespace sw {

namespace ek {
constexpr int NT = 256;   // threads per CTA: stage-in / write-back by all, the levels by the first LT
constexpr int LT = 64;    // the levels: one thread per box column (T0 <= 64)
}

struct Eik2Args {
    Geo G;
    int base;
    double h;
    const double *uo;   // padded u_old
    const double *S;    // padded slowness (> 0 on the domain)
    double *un;         // padded u_new
};

__device__ __forceinline__ double eik_inf() { return __longlong_as_double(0x7ff0000000000000LL); }

// Godunov solution (R-E1), the oracle's eik_godunov operation by operation
__device__ __forceinline__ double eik_godunov_d(double a, double b, double fh) {
    const double m = a < b ? a : b;
    if (m == eik_inf()) return m;
    if (fabs(__dsub_rn(a, b)) >= fh) return __dadd_rn(m, fh);
    const double d = __dsub_rn(a, b);
    const double disc = fma(-d, d, __dmul_rn(2.0, __dmul_rn(fh, fh)));
    return __dmul_rn(0.5, __dadd_rn(__dadd_rn(a, b), __dsqrt_rn(disc)));
}

// The same value without branches (the start-face chains, where the two candidates of a pair are
// independent and should overlap): every operand the oracle's eik_godunov would use is computed
// and the result selected.  The square root's argument is clamped to >= fh^2 / 4 so that it is
// always a positive normal number (no slow path); wherever its value is selected, |a - b| < fh and
// disc = 2 fh^2 - (a - b)^2 > fh^2, so the clamp never changes it.
__device__ __forceinline__ double eik_godunov_bf(double a, double b, double fh) {
    const double m = a < b ? a : b;
    const double d = __dsub_rn(a, b);
    const double fhfh = __dmul_rn(fh, fh);
    const double disc = fma(-d, d, __dmul_rn(2.0, fhfh));
    const double sq = __dsqrt_rn(fmax(disc, __dmul_rn(0.25, fhfh)));
    const double t2 = __dmul_rn(0.5, __dadd_rn(__dadd_rn(a, b), sq));
    const double r = fabs(d) >= fh ? __dadd_rn(m, fh) : t2;
    return m == eik_inf() ? m : r;
}

inline size_t eik2_smem(const Geo &G) {
    return sizeof(double) * ((size_t)(G.T[0] + 4) * (G.T[1] + 4) + (size_t)(G.T[0] + 1) * (G.T[1] + 1));
}

inline bool eik2_supported(const Geo &G) {
    return G.dim == 2 && G.T[0] <= 64 && G.T[1] <= 64 && eik2_smem(G) <= 227 * 1024;
}

#ifndef SW_EK_AHEAD
#define SW_EK_AHEAD 333
#endif
__global__ void __launch_bounds__(ek::NT, 3) k_eik2(Eik2Args A) {
    extern __shared__ __align__(16) double esm[];
    SW_JITTER_POINT();
    const Geo &G = A.G;
    const int T0 = G.T[0], T1 = G.T[1];
    const int WX = T0 + 4, FX = T0 + 1;
    double *const U = esm;                          // local [-2, T + 2) per axis
    double *const F = esm + WX * (T1 + 4);          // local [-1, T) per axis
    const int tx = blockIdx.x % G.nt[0], ty = blockIdx.x / G.nt[0];
    const int64_t R0 = tx, R1 = ty + G.toff[1];
    const int sx = ((A.base >> 0) & 1) ^ (int)(R0 & 1);
    const int sy = ((A.base >> 1) & 1) ^ (int)(R1 & 1);
    const bool cx = sx ? (R0 < G.ntg[0] - 1) : (R0 > 0);
    const bool cy = sy ? (R1 < G.ntg[1] - 1) : (R1 > 0);
    const int64_t X0 = R0 * T0, Y0 = R1 * T1;       // global min corner of the box
    auto gxo = [&](int lx) { return X0 + (sx ? T0 - 1 - lx : lx); };
    auto gyo = [&](int ly) { return Y0 + (sy ? T1 - 1 - ly : ly); };
    auto uw = [&](int lx, int ly) -> double & { return U[(ly + 2) * WX + (lx + 2)]; };
    auto fw = [&](int lx, int ly) -> double { return F[(ly + 1) * FX + (lx + 1)]; };
    SW_TMARK(t_start);
    // ---- stage in (old values, +inf outside the domain; slowness of the active region): warp w
    //      takes local rows w, w + 8, ..., lanes along x (consecutive addresses in either direction)
    int finite = 0;   // some old value of the window is finite
    {
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        const int nrow = T1 + 4;
#pragma unroll 2
        for (int r = warp; r < nrow; r += ek::NT / 32) {
            const int ly = r - 2;
            const int64_t gy = gyo(ly);
            const bool yin = gy >= 0 && gy < G.ng[1];
            const bool yact = ly >= -1 && ly < T1;
            const int64_t rowi = yin ? gidx(G, 0, gy, 0) : 0;
            double uv[3], sv[3];
#pragma unroll
            for (int c = 0; c < 3; ++c) {                  // lx = lane + 32 c - 2 < T0 + 2 <= 68 < 96
                const int lx = lane + 32 * c - 2;
                const int64_t gx = gxo(lx);
                const bool in = yin && lx < T0 + 2 && gx >= 0 && gx < G.ng[0];
                const bool act = yact && lx >= -1 && lx < T0;
                uv[c] = in ? __ldg(A.uo + rowi + gx) : eik_inf();
                sv[c] = (in && act) ? __ldg(A.S + rowi + gx) : 1.0;
            }
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const int lx = lane + 32 * c - 2;
                if (lx < T0 + 2) U[r * WX + (lx + 2)] = uv[c];
                finite |= uv[c] != eik_inf();
                if (yact && lx >= -1 && lx < T0) F[(ly + 1) * FX + (lx + 1)] = sv[c];
            }
        }
    }
    // a box whose whole window is +inf (not reached by the front yet) stays +inf: every Godunov
    // update of it sees +inf neighbours only (R-E1: u = +inf if min(a, b) = +inf), so it is copied
    // through unchanged -- exactly the oracle's result
    const bool reached = __syncthreads_or(finite);
    SW_TMARK(t_staged);
    SW_TADD(0, t_start, t_staged);
    if (!reached) {
        for (int e = threadIdx.x; e < T0 * T1; e += ek::NT) {
            const int lx = e % T0, ly = e / T0;
            A.un[gidx(G, gxo(lx), gyo(ly), 0)] = eik_inf();
        }
        SW_TADD(5, 0, 1);
        return;
    }
    if (threadIdx.x >= ek::LT) {           // the other warps rejoin for the write-back
#if SW_EK_AHEAD > 0
        {   // look-ahead: the lines of the box SW_EK_AHEAD launches later (u window and slowness,
            // clamped to the domain) into L2 while this box runs its chains and fronts
            const int64_t nb = (int64_t)blockIdx.x + SW_EK_AHEAD;
            if (nb < (int64_t)gridDim.x) {
                const int64_t nX0 = (nb % G.nt[0]) * T0 - 2, nY0 = (nb / G.nt[0] + G.toff[1]) * T1 - 2;
                const int NL = (T0 + 4 + 15) / 16 + 1;
                for (int e = threadIdx.x - ek::LT; e < (T1 + 4) * NL * 2; e += ek::NT - ek::LT) {
                    const int a = e & 1, q = e >> 1;
                    int64_t gx = nX0 + 16 * (q % NL), gy = nY0 + q / NL;
                    gx = gx < 0 ? 0 : (gx >= G.ng[0] ? G.ng[0] - 1 : gx);
                    gy = gy < 0 ? 0 : (gy >= G.ng[1] ? G.ng[1] - 1 : gy);
                    asm volatile("prefetch.global.L2 [%0];" ::"l"((a ? A.S : A.uo) + gidx(G, gx, gy, 0)));
                }
            }
        }
#endif
        __syncthreads();
        for (int e = threadIdx.x; e < T0 * T1; e += ek::NT) {
            const int lx = e % T0, ly = e / T0;
            A.un[gidx(G, gxo(lx), gyo(ly), 0)] = uw(lx, ly);
        }
        return;
    }
    const int t = threadIdx.x;
    // a node outside every coupled set: its window neighbours are new on its start side, old
    // elsewhere (in place, in a causal order), exactly the oracle's values
    auto single_upd = [&](int x, int y) {
        const double a = fmin(uw(x - 1, y), uw(x + 1, y)), b = fmin(uw(x, y - 1), uw(x, y + 1));
        const double ub = eik_godunov_d(a, b, __dmul_rn(fw(x, y), A.h));
        const double uo = uw(x, y);
        uw(x, y) = uo < ub ? uo : ub;
    };
    // candidate of member (px, py) with member (ox, oy) at value ov (+inf: unfixed)
    auto cand = [&](int px, int py, int ox, int oy, double ov) {
        const double w0 = (px - 1 == ox && py == oy) ? ov : uw(px - 1, py);
        const double w1 = (px + 1 == ox && py == oy) ? ov : uw(px + 1, py);
        const double v0 = (px == ox && py - 1 == oy) ? ov : uw(px, py - 1);
        const double v1 = (px == ox && py + 1 == oy) ? ov : uw(px, py + 1);
        const double ub = eik_godunov_d(fmin(w0, w1), fmin(v0, v1), __dmul_rn(fw(px, py), A.h));
        const double uo = uw(px, py);
        return uo < ub ? uo : ub;
    };
    // a pair across one coupled start face, ordered fixing written out (R-E3): both candidates
    // with the other member at +inf, the smaller (ties: lower global index) is fixed, the other
    // recomputed with it
    auto pairfix = [&](int x, int y, bool xf) {
        const int qx = xf ? -1 : x, qy = xf ? y : -1;
        const double cp = cand(x, y, qx, qy, eik_inf()), cq = cand(qx, qy, x, y, eik_inf());
        const int64_t gp = gyo(y) * G.ng[0] + gxo(x), gq = gyo(qy) * G.ng[0] + gxo(qx);
        const bool pfirst = gp < gq ? !(cq < cp) : (cp < cq);
        // the other member recomputed with the fixed one (one call with selected arguments, so
        // that the two chain lanes stay converged)
        const double fv = pfirst ? cp : cq;
        const double ov = pfirst ? cand(qx, qy, x, y, fv) : cand(x, y, qx, qy, fv);
        uw(x, y) = pfirst ? fv : ov;
        uw(qx, qy) = pfirst ? ov : fv;
    };
    // ---- the corner set, then the two start-face chains (row 0 with its partner row, column 0
    //      with its partner column), then the rest of the box level by level.  Any causal order
    //      gives the oracle's values (every node reads new values only on its start side); the
    //      chains first leave uniform single-node levels (no divergent set solves inside them).
    if (cx && cy && t < 32) {
        // the corner set (4 members), ordered fixing by lanes 0..3 of the warp: lane m owns member
        // (-(m & 1), -(m >> 1)) in local coordinates, whose member neighbours are lanes m ^ 1 (along
        // x) and m ^ 2 (along y), the other two neighbours come from the window.  Per round every
        // unfixed member's candidate (members at their fixed value or +inf), then the smallest
        // candidate by shuffles, ties to the lowest global index (the oracle scans the members in
        // ascending global order and keeps the first minimum); it is fixed.  (The other lane
        // groups of the warp compute the same and store nothing.)
        const int m = t & 3;
        const int mlx = -(m & 1), mly = -(m >> 1);
        const double xw = uw(mlx ? -2 : 1, mly), yw = uw(mlx, mly ? -2 : 1);
        const double uo = uw(mlx, mly), fh = __dmul_rn(fw(mlx, mly), A.h);
        const long long gi = (long long)(gyo(mly) * G.ng[0] + gxo(mlx));
        bool fixed = false;
        double val = eik_inf();
        for (int round = 0; round < 4; ++round) {
            const double mine = fixed ? val : eik_inf();
            const double xv = __shfl_xor_sync(0xffffffffu, mine, 1), yv = __shfl_xor_sync(0xffffffffu, mine, 2);
            const double ub = eik_godunov_d(xv < xw ? xv : xw, yv < yw ? yv : yw, fh);
            const double c = uo < ub ? uo : ub;
            double kc = fixed ? eik_inf() : c;
            long long kg = fixed ? 0x7fffffffffffffffLL : gi;
#pragma unroll
            for (int o = 1; o <= 2; o <<= 1) {
                const double oc = __shfl_xor_sync(0xffffffffu, kc, o);
                const long long og = __shfl_xor_sync(0xffffffffu, kg, o);
                const bool take = oc < kc || (oc == kc && og < kg);
                kc = take ? oc : kc;
                kg = take ? og : kg;
            }
            if (!fixed && kg == gi) {
                fixed = true;
                val = c;
            }
        }
        if (t < 4) uw(mlx, mly) = val;
    } else if (t == 0 && !(cx && cy)) {
        if (cx || cy) {
            pairfix(0, 0, cx);
        } else {
            single_upd(0, 0);
        }
    }
    __syncwarp();
    SW_JITTER_POINT();
    if (t < 2) {
        // lane 0: row 0 with the partner row (k, -1); lane 1: column 0 with the partner column
        // (-1, k); in step and branch-free: along the chain the member's and the partner's previous
        // values stay in registers (their west / south new neighbour), the old neighbours come from
        // the window (loaded a step ahead), the pair is solved by ordered fixing as pairfix does --
        // both candidates with the other member at +inf, the smaller fixed (its member order is
        // fixed per chain: the partner is first iff the box starts at the low end of the coupled
        // axis), the other recomputed by one Godunov update with selected operands.  Along an
        // uncoupled face the partner line lies outside the domain (+inf in the window), and the
        // plain update is the own candidate with the partner at +inf.
        const bool row = t == 0;
        const bool cpl = row ? cy : cx;
        const int len = row ? T0 : T1;
        const bool pfix = row ? (sy == 0) : (sx == 0);           // partner before own in global order
        // node k of the chain, offset o across the face (o = 0 own line, -1 partner line, +1 the
        // line after own, -2 the line beyond the partner)
        const int sk = row ? 1 : WX, so = row ? WX : 1;
        const double *const u0 = U + 2 * WX + 2;                 // local (0, 0)
        const double *const f0 = F + FX + 1;
        const int fk = row ? 1 : FX, fo = row ? FX : 1;
        double po = u0[0], pq = u0[-so];                          // the corner's results
        auto ld = [&](int k, double &uo_o, double &e_o, double &n_o, double &fh_o, double &uo_q, double &e_q,
                      double &s_q, double &fh_q) {
            const int kk = k < len ? k : len - 1;
            uo_o = u0[kk * sk]; e_o = u0[(kk + 1) * sk]; n_o = u0[kk * sk + so];
            uo_q = u0[kk * sk - so]; e_q = u0[(kk + 1) * sk - so]; s_q = u0[kk * sk - 2 * so];
            fh_o = __dmul_rn(f0[kk * fk], A.h);
            fh_q = __dmul_rn(f0[kk * fk - fo], A.h);   // (outside the domain: slowness 1, never used)
        };
        double uo_o, e_o, n_o, fh_o, uo_q, e_q, s_q, fh_q;
        ld(1, uo_o, e_o, n_o, fh_o, uo_q, e_q, s_q, fh_q);
        const double inf = eik_inf();
        for (int k = 1; k < len; ++k) {
            const double c_uo_o = uo_o, c_e_o = e_o, c_n_o = n_o, c_fh_o = fh_o;
            const double c_uo_q = uo_q, c_e_q = e_q, c_s_q = s_q, c_fh_q = fh_q;
            ld(k + 1, uo_o, e_o, n_o, fh_o, uo_q, e_q, s_q, fh_q);
            // own: W new (po), E old, across the face (vq), N old; partner: W new (pq), E old, S old,
            // across the face (vo)  (for the column chain the sides are swapped, and fmin is symmetric)
            const double a_o = fmin(po, c_e_o), a_q = fmin(pq, c_e_q);
            const double bo = eik_godunov_bf(a_o, fmin(inf, c_n_o), c_fh_o);
            const double bq = eik_godunov_bf(a_q, fmin(c_s_q, inf), c_fh_q);
            const double co = c_uo_o < bo ? c_uo_o : bo, cq = c_uo_q < bq ? c_uo_q : bq;
            const bool ofirst = pfix ? (co < cq) : !(cq < co);   // ties: the lower global index
            const double fv = ofirst ? co : cq;
            // the other member with the fixed one: cand_q(fv) if own is fixed, else cand_o(fv)
            const double ra = ofirst ? a_q : a_o;
            const double rb = ofirst ? fmin(c_s_q, fv) : fmin(fv, c_n_o);
            const double rfh = ofirst ? c_fh_q : c_fh_o, ruo = ofirst ? c_uo_q : c_uo_o;
            const double ub = eik_godunov_bf(ra, rb, rfh);
            const double ov = ruo < ub ? ruo : ub;
            const double res_o = cpl ? (ofirst ? fv : ov) : co;
            const double res_q = ofirst ? ov : fv;
            (row ? uw(k, 0) : uw(0, k)) = res_o;
            if (cpl) (row ? uw(k, -1) : uw(-1, k)) = res_q;
            po = res_o;
            pq = res_q;
        }
    }
    __syncwarp();
    SW_TMARK(t_chains);
    asm volatile("bar.sync 1, %0;" ::"r"(ek::LT) : "memory");   // the level threads only
    SW_JITTER_POINT();
    SW_TADD(1, t_staged, t_chains);
    for (int d = 2; d <= (T0 - 1) + (T1 - 1); ++d) {
        const int x = t, y = d - t;
        if (x >= 1 && x < T0 && y >= 1 && y < T1) single_upd(x, y);
        asm volatile("bar.sync 1, %0;" ::"r"(ek::LT) : "memory");
        SW_JITTER_POINT();
    }
    SW_TMARK(t_levels);
    SW_TADD(2, t_chains, t_levels);
    SW_TADD(5, 0, 1);
    __syncthreads();                          // with the waiting warps
    // ---- write-back of the box
    for (int e = threadIdx.x; e < T0 * T1; e += ek::NT) {
        const int lx = e % T0, ly = e / T0;
        A.un[gidx(G, gxo(lx), gyo(ly), 0)] = uw(lx, ly);
    }
}

inline cudaError_t launch_eik2(const Eik2Args &A, cudaStream_t s) {
    const size_t sm = eik2_smem(A.G);
    static size_t attr = 0;
    if (sm > attr) {
        cudaFuncSetAttribute(k_eik2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        attr = sm;
    }
    const unsigned tiles = (unsigned)((int64_t)A.G.nt[0] * A.G.nt[1]);
    k_eik2<<<tiles, ek::NT, sm, s>>>(A);
    return cudaGetLastError();
}

// number of interior nodes where a != b (the last eikonal pass changed them), per-CTA partials
__global__ void k_count_ne(Geo G, const double *a, const double *b, double *partial) {
    __shared__ double sh[8];
    const int64_t N = G.n[0] * G.n[1] * G.n[2];
    double c = 0.0;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < N; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i0 = t % G.n[0], r = t / G.n[0];
        const int64_t i = G.origin + i0 + G.P0 * (r % G.n[1]) + G.P01 * (r / G.n[1]);
        c += (a[i] != b[i]) ? 1.0 : 0.0;
    }
    for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += sh[w];
        partial[2 * blockIdx.x] = s;        // (count, 0): a double-double pair, exact below 2^53
        partial[2 * blockIdx.x + 1] = 0.0;
    }
}

}  // namespace sw
