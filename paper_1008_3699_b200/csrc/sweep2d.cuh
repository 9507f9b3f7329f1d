// sweep2d.cuh -- specialised 2D decomposed SOR sweep for 64 x 64 boxes (sm_100a).
//
// One CTA = one warp = one box (SURVEY §7 "2D kernel sketch").
//  * Stage-in: one TMA tiled load of the 68 x 68 window of x_old (box + 2-node halo,
//    PAPER:828-833), one of the 64 x 64 b tile (and two 68 x 68 face windows for variable
//    coefficients); the few right-hand sides of the partner nodes across the start faces
//    come in by plain loads.  All land in shared memory, completion on an mbarrier.
//  * Wavefront: the box is reflected so its start corner is local (0,0).  Lane l owns
//    local rows l (band 0) and l+32 (band 1); at step s it updates local node
//    (c = s - l - 64 band, row).  The implicit west value is the lane's own previous
//    result (register), the implicit south value arrives from lane l-1 by warp shuffle
//    (band 1, lane 0: from shared memory), explicit east/north values are old values still
//    in shared memory.  159 steps, one __syncwarp per step, updates in place.
//  * Coupled systems: at step 0 lane 0 solves the start-corner set (4 x 4 if both start
//    faces are coupled, eq 2d:sor4b4, else 2 x 2 / 1 x 1); lane 0 carries the y-start-face
//    chain of 2 x 2 systems along row 0 (eq 2d:sor2b2), lane t solves the x-start-face pair
//    of row t at column 0.  Elimination order and fused operations are those of the oracle
//    (DESIGN R-7, R-8), so results are bitwise identical.
//  * Write-back: 64 one-row bulk copies (cp.async.bulk) of the updated interior to x_new.
#pragma once
#include <cuda.h>

#include "common.cuh"
#include "tma.cuh"

namespace sw {

constexpr int T2 = 64;    // box edge
constexpr int WW = 68;    // window edge (box + 2 halo each side)
constexpr int WSZ = WW * WW;

struct Maps2d {
    CUtensorMap x[2], b, f0, f1;
    bool ok = false;
};

struct Sweep2dArgs {
    Geo G;
    int base;
    double omega[4];
    const double *b;    // padded b (partner right-hand sides)
    double *xnew;       // padded x_new
    int *flag;
};

template <bool FACES>
__host__ __device__ constexpr size_t sweep2d_smem() {
    return sizeof(double) * (WSZ + T2 * T2 + 2 * T2 + 8 + (FACES ? 2 * WSZ : 0)) + 16;
}

// face coefficient between window columns a and a+1 (row wr) / rows a and a+1 (column wc)
template <bool FACES>
__device__ __forceinline__ double fxb(const double *fx, int wr, int a) {
    if constexpr (FACES) return fx[wr * WW + a + 1];
    return 1.0;
}
template <bool FACES>
__device__ __forceinline__ double fyb(const double *fy, int a, int wc) {
    if constexpr (FACES) return fy[(a + 1) * WW + wc];
    return 1.0;
}

// a_P of window node (wr, wc): x-, x+, y-, y+, then beta (DESIGN R-7)
template <bool FACES>
__device__ __forceinline__ double ap_w(const double *fx, const double *fy, int wr, int wc, double beta) {
    double s = 0.0;
    s += fxb<FACES>(fx, wr, wc - 1);
    s += fxb<FACES>(fx, wr, wc);
    s += fyb<FACES>(fy, wr - 1, wc);
    s += fyb<FACES>(fy, wr, wc);
    return s + beta;
}

// Gaussian elimination without pivoting, reciprocal pivots, fused updates: identical to
// the oracle's ge_solve (DESIGN R-8).
template <int K>
__device__ __forceinline__ void ge_small(double (&M)[K][K], double (&rhs)[K], double (&u)[K], int *flag) {
    double inv[K];
#pragma unroll
    for (int p = 0; p < K; ++p) {
        double piv = M[p][p];
        if (!(fabs(piv) >= 1e-14)) atomicOr(flag, 1);
        inv[p] = 1.0 / piv;
#pragma unroll
        for (int q = p + 1; q < K; ++q) {
            double l = M[q][p] * inv[p];
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

// 2x2 coupled pair in member order (a, b): rows u_a - m_ab u_b = r_a, u_b - m_ba u_a = r_b.
__device__ __forceinline__ void pair_solve(double ra, double rb, double mab, double mba, double &ua, double &ub,
                                           int *flag) {
    double M11 = fma(mba, -mab, 1.0);
    double r1 = fma(mba, ra, rb);
    if (!(fabs(M11) >= 1e-14)) atomicOr(flag, 1);
    double inv1 = 1.0 / M11;
    ub = r1 * inv1;
    ua = fma(mab, ub, ra) * 1.0;
}

template <bool FACES>
__global__ void __launch_bounds__(32, FACES ? 1 : 3)
    k_sweep2d(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmb,
              const __grid_constant__ CUtensorMap tmf0, const __grid_constant__ CUtensorMap tmf1, Sweep2dArgs A) {
    extern __shared__ __align__(128) double sm[];
    double *xw = sm;                              // x window, global orientation
    double *bt = xw + WSZ;                        // b tile, global orientation
    double *fx = bt + T2 * T2;                    // F_x window (FACES); every TMA target 128-B aligned
    double *fy = fx + WSZ;                        // F_y window (FACES)
    double *bpx = FACES ? fy + WSZ : fx;          // b of the x-partners (-1, t), by local t
    double *bpy = bpx + T2;                       // b of the y-partners (c, -1), by local c; [64] = corner
    __shared__ uint64_t bar;

    const Geo &G = A.G;
    const int lane = threadIdx.x;
    const int tx = blockIdx.x % G.nt[0];
    const int ty = blockIdx.x / G.nt[0];
    const int64_t R0 = tx, R1 = ty + G.toff[1];
    const int x0 = tx * T2;                       // global = local along x
    const int y0l = ty * T2;                      // slab-local
    const int sx = ((A.base >> 0) & 1) ^ (int)(R0 & 1);
    const int sy = ((A.base >> 1) & 1) ^ (int)(R1 & 1);
    const bool cx = sx ? (R0 < G.ntg[0] - 1) : (R0 > 0);
    const bool cy = sy ? (R1 < G.ntg[1] - 1) : (R1 > 0);
    const int bits = sx | (sy << 1);
    const double beta = G.beta;

    if (lane == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    __syncwarp();
    if (lane == 0) {
        uint32_t bytes = sizeof(double) * (WSZ + T2 * T2 + (FACES ? 2 * WSZ : 0));
        mbar_expect_tx(&bar, bytes);
        tma_load_2d(xw, &tmx, x0, y0l, &bar);
        tma_load_2d(bt, &tmb, x0 + 2, y0l + 2, &bar);
        if constexpr (FACES) {
            tma_load_2d(fx, &tmf0, x0, y0l, &bar);
            tma_load_2d(fy, &tmf1, x0, y0l, &bar);
        }
    }
    // right-hand sides of the partner nodes (padded b: padded (gx+2, local gy+2))
    {
        const int pxw = sx ? x0 + T2 : x0 - 1;          // global x of local column -1
        const int pyl = sy ? y0l + T2 : y0l - 1;        // slab-local y of local row -1
        for (int i = lane; i < T2; i += 32) {
            int gyl = sy ? y0l + T2 - 1 - i : y0l + i;
            int gx = sx ? x0 + T2 - 1 - i : x0 + i;
            bpx[i] = cx ? A.b[(int64_t)(gyl + 2) * G.P0 + pxw + 2] : 0.0;
            bpy[i] = cy ? A.b[(int64_t)(pyl + 2) * G.P0 + gx + 2] : 0.0;
        }
        if (lane == 0) bpy[T2] = (cx && cy) ? A.b[(int64_t)(pyl + 2) * G.P0 + pxw + 2] : 0.0;
    }
    mbar_wait(&bar, 0);
    __syncwarp();

    // local -> window maps
    const int dX = sx ? -1 : 1;              // window column step for local +x
    const int dY = sy ? -1 : 1;              // window row step for local +y
    auto WX = [&](int c) { return 2 + (sx ? T2 - 1 - c : c); };
    auto WY = [&](int t) { return 2 + (sy ? T2 - 1 - t : t); };
    // face between window nodes (r,c) and (r, c+d) / (r+d, c)
    auto cxw = [&](int r, int c, int d) { return fxb<FACES>(fx, r, d > 0 ? c : c - 1); };
    auto cyw = [&](int r, int c, int d) { return fyb<FACES>(fy, d > 0 ? r : r - 1, c); };

    const double w_own = A.omega[bits], w_px = A.omega[bits ^ 1], w_py = A.omega[bits ^ 2],
                 w_pd = A.omega[bits ^ 3];
    const double omw = 1.0 - w_own;
    // Poisson: constant alpha
    const double ap_c = ap_w<false>(nullptr, nullptr, 2, 2, beta);
    const double al_c = w_own / ap_c;

    // per-node right-hand side r0 = fma(alpha, b + explicit terms, (1-w) u_old) at window (r, c)
    // with explicit neighbours at local +x (d = dX) and local +y (dY) unless flipped for partners
    auto node_r0 = [&](int r, int c, int ex, int ey, double w, double bval, double &al) {
        double ap = ap_w<FACES>(fx, fy, r, c, beta);
        al = w / ap;
        double e = fma(cxw(r, c, ex), xw[r * WW + c + ex], bval);
        e = fma(cyw(r, c, ey), xw[(r + ey) * WW + c], e);
        return fma(al, e, (1.0 - w) * xw[r * WW + c]);
    };

    double u = 0.0, par = 0.0;       // last own value, last x-partner value (shuffled to lane+1)
    double Wown = 0.0, Wpy = 0.0;     // west (own previous) value; y-chain partner previous value (lane 0)
    double Eprev = 0.0;
    for (int s = 0; s < 2 * T2 + 31; ++s) {
        const double Ssh = __shfl_up_sync(0xffffffffu, u, 1);
        const double Psh = __shfl_up_sync(0xffffffffu, par, 1);
        const int k = s - lane;
        if (k >= 0 && k < 2 * T2) {
            const int band = k >> 6;
            const int c = k & (T2 - 1);
            const int t = band * 32 + lane;
            const int r = WY(t), wc = WX(c);
            const double uo = (c == 0) ? xw[r * WW + wc] : Eprev;
            const double E = xw[r * WW + wc + dX];
            const double N = xw[(r + dY) * WW + wc];
            const double bv = bt[(sy ? T2 - 1 - t : t) * T2 + (sx ? T2 - 1 - c : c)];
            double S;
            if (lane != 0) S = Ssh;
            else if (band == 1) S = xw[(r - dY) * WW + wc];
            else S = 0.0;   // row 0: boundary or coupled partner (handled below)
            if (c == 0) Wown = 0.0;
            double al, r0;
            if constexpr (FACES) {
                r0 = node_r0(r, wc, dX, dY, w_own, bv, al);
            } else {
                al = al_c;
                double e = fma(1.0, E, bv);
                e = fma(1.0, N, e);
                r0 = fma(al, e, omw * uo);
            }
            const double mW = al * cxw(r, wc, -dX);
            const double mS = al * cyw(r, wc, -dY);
            if (c == 0 && t == 0) {
                // ---- start corner (lane 0, step 0)
                const int rp = r - dY, cp = wc - dX;    // window row of local -1, column of local -1
                if (cx && cy) {
                    // members in ascending global index: rows (low y first), then columns (low x first)
                    int mr[4], mc[4], mb[4];
                    const int rlo = sy ? r : rp, rhi = sy ? rp : r, clo = sx ? wc : cp, chi = sx ? cp : wc;
                    const int rr_[4] = {rlo, rlo, rhi, rhi}, cc_[4] = {clo, chi, clo, chi};
                    double M[4][4], rhs[4], uu[4];
                    for (int m = 0; m < 4; ++m) {
                        mr[m] = rr_[m];
                        mc[m] = cc_[m];
                        // local coordinates of member m: -1 where the window coordinate is the partner's
                        const bool lx = (mc[m] == cp), ly = (mr[m] == rp);
                        mb[m] = bits ^ (lx ? 1 : 0) ^ (ly ? 2 : 0);
                    }
                    for (int m = 0; m < 4; ++m) {
                        for (int q = 0; q < 4; ++q) M[m][q] = (m == q) ? 1.0 : 0.0;
                        const bool lx = (mc[m] == cp), ly = (mr[m] == rp);
                        // explicit sides: own box local +x/+y; flipped for partner boxes
                        const int ex = lx ? -dX : dX, ey = ly ? -dY : dY;
                        const double w = A.omega[mb[m]];
                        const double bval = (lx && ly) ? bpy[T2] : (lx ? bpx[0] : (ly ? bpy[0] : bv));
                        double alm;
                        double r0m;
                        if constexpr (FACES) {
                            r0m = node_r0(mr[m], mc[m], ex, ey, w, bval, alm);
                        } else {
                            alm = w / ap_c;
                            double e = fma(1.0, xw[mr[m] * WW + mc[m] + ex], bval);
                            e = fma(1.0, xw[(mr[m] + ey) * WW + mc[m]], e);
                            r0m = fma(alm, e, (1.0 - w) * xw[mr[m] * WW + mc[m]]);
                        }
                        rhs[m] = r0m;
                        // coupling to the x-flip and y-flip members
                        const int qx = m ^ 1, qy = m ^ 2;
                        M[m][qx] = -(alm * cxw(mr[m], mc[m], mc[qx] - mc[m]));
                        M[m][qy] = -(alm * cyw(mr[m], mc[m], mr[qy] - mr[m]));
                    }
                    ge_small<4>(M, rhs, uu, A.flag);
                    for (int m = 0; m < 4; ++m) xw[mr[m] * WW + mc[m]] = uu[m];
                    int own = 0, px = 0, py = 0;
                    for (int m = 0; m < 4; ++m) {
                        if (mr[m] == r && mc[m] == wc) own = m;
                        if (mr[m] == r && mc[m] == cp) px = m;
                        if (mr[m] == rp && mc[m] == wc) py = m;
                    }
                    u = uu[own];
                    par = uu[px];
                    Wpy = uu[py];
                } else if (cx) {
                    // pair (own, x-partner); neither has an external dependency (boundary below)
                    double alp;
                    double r0p;
                    if constexpr (FACES) {
                        r0p = node_r0(r, cp, -dX, dY, w_px, bpx[0], alp);
                    } else {
                        alp = w_px / ap_c;
                        double e = fma(1.0, xw[r * WW + cp - dX], bpx[0]);
                        e = fma(1.0, xw[(r + dY) * WW + cp], e);
                        r0p = fma(alp, e, (1.0 - w_px) * xw[r * WW + cp]);
                    }
                    const double r0o = fma(mS, 0.0, r0);
                    const double r0pp = fma(alp * cyw(r, cp, -dY), 0.0, r0p);
                    const double mop = al * cxw(r, wc, -dX), mpo = alp * cxw(r, cp, dX);
                    double uo_, up_;
                    if (sx == 0) pair_solve(r0pp, r0o, mpo, mop, up_, uo_, A.flag);
                    else pair_solve(r0o, r0pp, mop, mpo, uo_, up_, A.flag);
                    u = uo_;
                    par = up_;
                    xw[r * WW + cp] = up_;
                } else if (cy) {
                    double alp;
                    double r0p;
                    if constexpr (FACES) {
                        r0p = node_r0(rp, wc, dX, -dY, w_py, bpy[0], alp);
                    } else {
                        alp = w_py / ap_c;
                        double e = fma(1.0, xw[rp * WW + wc + dX], bpy[0]);
                        e = fma(1.0, xw[(rp - dY) * WW + wc], e);
                        r0p = fma(alp, e, (1.0 - w_py) * xw[rp * WW + wc]);
                    }
                    const double r0o = fma(mW, 0.0, r0);
                    const double r0pp = fma(alp * cxw(rp, wc, -dX), 0.0, r0p);
                    const double mop = al * cyw(r, wc, -dY), mpo = alp * cyw(rp, wc, dY);
                    double uo_, up_;
                    if (sy == 0) pair_solve(r0pp, r0o, mpo, mop, up_, uo_, A.flag);
                    else pair_solve(r0o, r0pp, mop, mpo, uo_, up_, A.flag);
                    u = uo_;
                    Wpy = up_;
                    xw[rp * WW + wc] = up_;
                } else {
                    u = fma(mS, 0.0, fma(mW, 0.0, r0));
                }
                (void)w_pd;
            } else if (c == 0 && cx) {
                // ---- x-start-face pair of row t: own (0,t) & partner (-1,t)   (eq 2d:sor2b2)
                const int cp = wc - dX;
                const double Pp = (lane != 0) ? Psh : xw[(r - dY) * WW + cp];   // partner (-1, t-1), new
                double alp;
                double r0p;
                if constexpr (FACES) {
                    r0p = node_r0(r, cp, -dX, dY, w_px, bpx[t], alp);
                } else {
                    alp = w_px / ap_c;
                    double e = fma(1.0, xw[r * WW + cp - dX], bpx[t]);
                    e = fma(1.0, xw[(r + dY) * WW + cp], e);
                    r0p = fma(alp, e, (1.0 - w_px) * xw[r * WW + cp]);
                }
                const double ro = fma(mS, S, r0);
                const double rp_ = fma(alp * cyw(r, cp, -dY), Pp, r0p);
                const double mop = al * cxw(r, wc, -dX), mpo = alp * cxw(r, cp, dX);
                double uo_, up_;
                if (sx == 0) pair_solve(rp_, ro, mpo, mop, up_, uo_, A.flag);
                else pair_solve(ro, rp_, mop, mpo, uo_, up_, A.flag);
                u = uo_;
                par = up_;
                xw[r * WW + cp] = up_;
            } else if (t == 0 && cy) {
                // ---- y-start-face pair of column c: own (c,0) & partner (c,-1)
                const int rp = r - dY;
                double alp;
                double r0p;
                if constexpr (FACES) {
                    r0p = node_r0(rp, wc, dX, -dY, w_py, bpy[c], alp);
                } else {
                    alp = w_py / ap_c;
                    double e = fma(1.0, xw[rp * WW + wc + dX], bpy[c]);
                    e = fma(1.0, xw[(rp - dY) * WW + wc], e);
                    r0p = fma(alp, e, (1.0 - w_py) * xw[rp * WW + wc]);
                }
                const double ro = fma(mW, Wown, r0);
                const double rp_ = fma(alp * cxw(rp, wc, -dX), Wpy, r0p);
                const double mop = al * cyw(r, wc, -dY), mpo = alp * cyw(rp, wc, dY);
                double uo_, up_;
                if (sy == 0) pair_solve(rp_, ro, mpo, mop, up_, uo_, A.flag);
                else pair_solve(ro, rp_, mop, mpo, uo_, up_, A.flag);
                u = uo_;
                Wpy = up_;
                xw[rp * WW + wc] = up_;
            } else {
                // ---- interior node: implicit west (own register) then south (shuffle)
                u = fma(mS, S, fma(mW, Wown, r0));
            }
            xw[r * WW + wc] = u;
            Wown = u;
            Eprev = E;
        }
        __syncwarp();
    }

    // write back the 64 x 64 interior, one bulk copy per row
    fence_proxy_async_smem();
    __syncwarp();
    for (int rr = lane; rr < T2; rr += 32) {
        double *dst = A.xnew + (int64_t)(y0l + rr + 2) * G.P0 + (x0 + 2);
        bulk_store(dst, xw + (rr + 2) * WW + 2, T2 * sizeof(double));
    }
    bulk_commit();
    bulk_wait_read0();
}

inline bool sweep2d_supported(const Geo &G) {
    return G.dim == 2 && G.T[0] == T2 && G.T[1] == T2 && G.off[0] == 0 && (G.P0 % 2) == 0;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn get_encode() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (EncodeTiledFn)p;
    }
    return fn;
}

inline bool encode_2d(CUtensorMap *m, const double *base, int64_t pad0, int64_t pad1, int box0, int box1) {
    EncodeTiledFn enc = get_encode();
    if (!enc || !base) return false;
    cuuint64_t dims[2] = {(cuuint64_t)pad0, (cuuint64_t)pad1};
    cuuint64_t strides[1] = {(cuuint64_t)(pad0 * sizeof(double))};
    cuuint32_t box[2] = {(cuuint32_t)box0, (cuuint32_t)box1};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void *)base, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

inline bool make_maps2d(Maps2d &M, const double *x0, const double *x1, const double *b, const double *f0,
                        const double *f1, int64_t pad0, int64_t pad1) {
    M.ok = encode_2d(&M.x[0], x0, pad0, pad1, WW, WW) && encode_2d(&M.x[1], x1, pad0, pad1, WW, WW) &&
           encode_2d(&M.b, b, pad0, pad1, T2, T2);
    if (M.ok && f0) M.ok = encode_2d(&M.f0, f0, pad0, pad1, WW, WW) && encode_2d(&M.f1, f1, pad0, pad1, WW, WW);
    else if (M.ok) {
        M.f0 = M.x[0];
        M.f1 = M.x[0];
    }
    return M.ok;
}

inline cudaError_t launch_sweep2d(const Maps2d &M, int cur, const Geo &G, int base, const double *w8,
                                  const double *b, double *xn, int *flag, bool faces, cudaStream_t s) {
    Sweep2dArgs A;
    A.G = G;
    A.base = base;
    for (int i = 0; i < 4; ++i) A.omega[i] = w8[i];
    A.b = b;
    A.xnew = xn;
    A.flag = flag;
    unsigned tiles = (unsigned)((int64_t)G.nt[0] * G.nt[1]);
    if (faces) {
        size_t sm = sweep2d_smem<true>();
        cudaFuncSetAttribute(k_sweep2d<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k_sweep2d<true><<<tiles, 32, sm, s>>>(M.x[cur], M.b, M.f0, M.f1, A);
    } else {
        size_t sm = sweep2d_smem<false>();
        cudaFuncSetAttribute(k_sweep2d<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k_sweep2d<false><<<tiles, 32, sm, s>>>(M.x[cur], M.b, M.f0, M.f1, A);
    }
    return cudaGetLastError();
}

}  // namespace sw
