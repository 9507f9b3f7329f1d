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
// Thread 0 solves the corner set, then threads 0 and 1 run the two start-face chains (row 0 with
// its partner row, column 0 with its partner column: pairs by ordered fixing, or plain updates
// along an uncoupled face); then level d = x + y of the other own nodes: thread t < 64 takes node
// (t, d - t) directly from the window; results go in place (the window then holds new values on
// every node's start side and old values on its end side, exactly the split the method
// prescribes); a named barrier of the 64 level threads per level; write-back by all threads.
#pragma once
#include "common.cuh"

namespace sw {

namespace ek {
constexpr int NT = 256;   // threads per CTA: stage-in / write-back by all, the levels by the first LT
constexpr int LT = 64;    // one thread per box column (T0 <= 64)
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

inline size_t eik2_smem(const Geo &G) {
    return sizeof(double) * ((size_t)(G.T[0] + 4) * (G.T[1] + 4) + (size_t)(G.T[0] + 1) * (G.T[1] + 1));
}

inline bool eik2_supported(const Geo &G) {
    return G.dim == 2 && G.T[0] <= ek::LT && G.T[1] <= ek::LT && eik2_smem(G) <= 227 * 1024;
}

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
                if (yact && lx >= -1 && lx < T0) F[(ly + 1) * FX + (lx + 1)] = sv[c];
            }
        }
    }
    __syncthreads();
    SW_TMARK(t_staged);
    SW_TADD(0, t_start, t_staged);
    if (threadIdx.x >= ek::LT) {           // the other warps rejoin for the write-back
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
    if (t == 0) {
        if (cx && cy) {
            // the corner set (4 members) in local coordinates, generic ordered fixing
            int mx[4] = {0, -1, 0, -1}, my[4] = {0, 0, -1, -1};
            constexpr int k = 4;
            // ascending global index (the oracle's member order; ties in the selection go to it)
            int64_t gi[4];
            for (int m = 0; m < k; ++m) gi[m] = gyo(my[m]) * G.ng[0] + gxo(mx[m]);
            for (int a1 = 1; a1 < k; ++a1)
                for (int b1 = a1; b1 > 0 && gi[b1 - 1] > gi[b1]; --b1) {
                    int64_t tg = gi[b1]; gi[b1] = gi[b1 - 1]; gi[b1 - 1] = tg;
                    int tt = mx[b1]; mx[b1] = mx[b1 - 1]; mx[b1 - 1] = tt;
                    tt = my[b1]; my[b1] = my[b1 - 1]; my[b1 - 1] = tt;
                }
            bool fixed[4] = {false, false, false, false};
            double val[4];
            for (int round = 0; round < k; ++round) {
                int best = -1;
                double cbest = 0.0;
                for (int m = 0; m < k; ++m) {
                    if (fixed[m]) continue;
                    // a neighbour that is a member: its fixed value or +inf; else the window
                    auto nb = [&](int lx, int ly) -> double {
                        for (int q = 0; q < k; ++q)
                            if (mx[q] == lx && my[q] == ly) return fixed[q] ? val[q] : eik_inf();
                        return uw(lx, ly);
                    };
                    const int px = mx[m], py = my[m];
                    const double w0 = nb(px - 1, py), w1 = nb(px + 1, py);
                    const double v0 = nb(px, py - 1), v1 = nb(px, py + 1);
                    // (the oracle visits the sides in global order -, +; min is order independent)
                    const double a = w0 < w1 ? w0 : w1, b = v0 < v1 ? v0 : v1;
                    const double ub = eik_godunov_d(a, b, __dmul_rn(fw(px, py), A.h));
                    const double uo = uw(px, py);
                    const double c = uo < ub ? uo : ub;
                    if (best < 0 || c < cbest) {
                        best = m;
                        cbest = c;
                    }
                }
                fixed[best] = true;
                val[best] = cbest;
            }
            for (int m = 0; m < k; ++m) uw(mx[m], my[m]) = val[m];
        } else if (cx || cy) {
            pairfix(0, 0, cx);
        } else {
            single_upd(0, 0);
        }
    }
    __syncwarp();
    if (t < 2) {
        // lane 0: row 0 with the partner row (k, -1); lane 1: column 0 with the partner column
        // (-1, k); in step, with the pair geometry written out: along the chain the member's and the
        // partner's previous values stay in registers (their west / south new neighbour), the old
        // neighbours come from the window, the pair is solved by ordered fixing as pairfix does
        // (its member order is fixed per chain: the partner is first iff the box starts at the low
        // end of the coupled axis)
        const bool row = t == 0;
        const bool cpl = row ? cy : cx;
        const int len = row ? T0 : T1;
        const bool pfix = row ? (sy == 0) : (sx == 0);           // partner before own in global order
        // window accessors in chain coordinates: node k of the chain, offset o across the face
        // (o = 0 own line, -1 partner line, +1 the line after own, -2 the line beyond the partner)
        auto cw = [&](int k, int o) -> double { return row ? uw(k, o) : uw(o, k); };
        auto cf = [&](int k, int o) -> double { return row ? fw(k, o) : fw(o, k); };
        double po = cw(0, 0), pq = cw(0, -1);                       // the corner's results
        const double inf = eik_inf();
        for (int k = 1; k < (T0 > T1 ? T0 : T1); ++k) {
            if (k < len) {
                const double uo_o = cw(k, 0), e_o = cw(k + 1, 0), n_o = cw(k, 1);
                const double fh_o = __dmul_rn(cf(k, 0), A.h);
                double res_o, res_q;
                if (cpl) {
                    const double uo_q = cw(k, -1), e_q = cw(k + 1, -1), s_q = cw(k, -2);
                    const double fh_q = __dmul_rn(cf(k, -1), A.h);
                    // chain-along pairs (the oracle's sides in global order are order independent: min)
                    auto cand_o = [&](double vq) {       // own: W new (po), E old, across the face vq, N old
                        const double ub = eik_godunov_d(fmin(po, e_o), fmin(vq, n_o), fh_o);
                        return uo_o < ub ? uo_o : ub;
                    };
                    auto cand_q = [&](double vo) {       // partner: W new (pq), E old, S old, across vo
                        const double ub = eik_godunov_d(fmin(pq, e_q), fmin(s_q, vo), fh_q);
                        return uo_q < ub ? uo_q : ub;
                    };
                    // (for the column chain "W/E" are the partner's and own's south / north sides and
                    //  "across" the west / east side: a = min over x, b = min over y either way,
                    //  and fmin is symmetric, so the same two mins result)
                    const double co = cand_o(inf), cq = cand_q(inf);
                    const bool ofirst = pfix ? (co < cq) : !(cq < co);   // ties: the lower global index
                    const double fv = ofirst ? co : cq;
                    const double ov = ofirst ? cand_q(fv) : cand_o(fv);
                    res_o = ofirst ? fv : ov;
                    res_q = ofirst ? ov : fv;
                    (row ? uw(k, -1) : uw(-1, k)) = res_q;
                } else {
                    const double ub = eik_godunov_d(fmin(po, e_o), fmin(cw(k, -1), n_o), fh_o);
                    res_o = uo_o < ub ? uo_o : ub;
                    res_q = pq;
                }
                (row ? uw(k, 0) : uw(0, k)) = res_o;
                po = res_o;
                pq = res_q;
            }
        }
    }
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
