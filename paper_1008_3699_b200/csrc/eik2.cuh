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
// Level d = x + y of the own nodes: thread t < 64 takes own node (t, d - t) -- directly from the
// window when it is in no coupled set, else with its partner layer by ordered fixing; results go
// in place (the window then holds new values on every node's start side and old values on its end
// side, exactly the split the method prescribes); a named barrier of the 64 level threads per
// level; write-back of the box by all threads.
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
    // ---- stage in (old values, +inf outside the domain; slowness of the active region)
#pragma unroll 4
    for (int e = threadIdx.x; e < WX * (T1 + 4); e += ek::NT) {
        const int lx = e % WX - 2, ly = e / WX - 2;
        const int64_t gx = gxo(lx), gy = gyo(ly);
        const bool in = gx >= 0 && gx < G.ng[0] && gy >= 0 && gy < G.ng[1];
        const bool act = lx >= -1 && lx < T0 && ly >= -1 && ly < T1;
        const int64_t gi = in ? gidx(G, gx, gy, 0) : 0;
        const double uv = in ? __ldg(A.uo + gi) : eik_inf();
        const double sv = (in && act) ? __ldg(A.S + gi) : 1.0;
        U[e] = uv;
        if (act) F[(ly + 1) * FX + (lx + 1)] = sv;
    }
    __syncthreads();
    if (threadIdx.x >= ek::LT) {           // the other warps rejoin for the write-back
        __syncthreads();
        for (int e = threadIdx.x; e < T0 * T1; e += ek::NT) {
            const int lx = e % T0, ly = e / T0;
            A.un[gidx(G, gxo(lx), gyo(ly), 0)] = uw(lx, ly);
        }
        return;
    }
    // ---- levels
    const int t = threadIdx.x;
    for (int d = 0; d <= (T0 - 1) + (T1 - 1); ++d) {
        const int x = t, y = d - t;
        const bool single = !((x == 0 && cx) || (y == 0 && cy));
        if (x < T0 && y >= 0 && y < T1 && single) {
            // a node outside every coupled set: its window neighbours are new on its start side,
            // old elsewhere (in place, level order), exactly the oracle's values
            const double a = fmin(uw(x - 1, y), uw(x + 1, y)), b = fmin(uw(x, y - 1), uw(x, y + 1));
            const double ub = eik_godunov_d(a, b, __dmul_rn(fw(x, y), A.h));
            const double uo = uw(x, y);
            uw(x, y) = uo < ub ? uo : ub;
        } else if (x < T0 && y >= 0 && y < T1 && !(x == 0 && y == 0 && cx && cy)) {
            // a pair across one coupled start face, ordered fixing written out (R-E3): both
            // candidates with the other member at +inf, the smaller (ties: lower global index) is
            // fixed, the other recomputed with it
            const bool xf = x == 0 && cx;
            const int qx = xf ? -1 : x, qy = xf ? y : -1;
            auto cand = [&](int px, int py, int ox, int oy, double ov) {
                const double w0 = (px - 1 == ox && py == oy) ? ov : uw(px - 1, py);
                const double w1 = (px + 1 == ox && py == oy) ? ov : uw(px + 1, py);
                const double v0 = (px == ox && py - 1 == oy) ? ov : uw(px, py - 1);
                const double v1 = (px == ox && py + 1 == oy) ? ov : uw(px, py + 1);
                const double ub = eik_godunov_d(fmin(w0, w1), fmin(v0, v1), __dmul_rn(fw(px, py), A.h));
                const double uo = uw(px, py);
                return uo < ub ? uo : ub;
            };
            const double cp = cand(x, y, qx, qy, eik_inf()), cq = cand(qx, qy, x, y, eik_inf());
            const int64_t gp = gyo(y) * G.ng[0] + gxo(x), gq = gyo(qy) * G.ng[0] + gxo(qx);
            const bool pfirst = gp < gq ? !(cq < cp) : (cp < cq);
            double up, uq;
            if (pfirst) {
                up = cp;
                uq = cand(qx, qy, x, y, up);
            } else {
                uq = cq;
                up = cand(x, y, qx, qy, uq);
            }
            uw(x, y) = up;
            uw(qx, qy) = uq;
        } else if (x < T0 && y >= 0 && y < T1) {
            // the corner set (4 members) in local coordinates, generic ordered fixing
            int mx[4], my[4], k = 1;
            mx[0] = x;
            my[0] = y;
            if (x == 0 && y == 0 && cx && cy) {
                mx[1] = -1; my[1] = 0; mx[2] = 0; my[2] = -1; mx[3] = -1; my[3] = -1;
                k = 4;
            } else if (x == 0 && cx) {
                mx[1] = -1; my[1] = y;
                k = 2;
            } else if (y == 0 && cy) {
                mx[1] = x; my[1] = -1;
                k = 2;
            }
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
        }
        asm volatile("bar.sync 1, %0;" ::"r"(ek::LT) : "memory");   // the level threads only
        SW_JITTER_POINT();
    }
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
