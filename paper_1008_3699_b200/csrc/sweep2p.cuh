// sweep2p.cuh -- 2D decomposed SOR sweep, constant coefficients (Poisson), 64 x 64 boxes,
// sm_100a.  Version 2 of the 2D kernel (the v1 kernel in sweep2d.cuh still serves the
// variable-coefficient case).
//
// One CTA = one warp = one box.  Six CTAs fit on an SM (36 KB of shared
// memory each).  Per box:
//  1. Stage-in: one TMA load of the 68 x 68 window of x_old (box + 2-node halo,
//     PAPER:828-833) into shared memory; the 64 rows of b are prefetched into L2 with bulk
//     prefetches and read back coalesced through a register ring.
//  2. Explicit parts (data parallel, coalesced): every owned node's
//        r0 = fma(w/a_P, (b + u_E) + u_N, (1-w) u)         (DESIGN R-7)
//     is written over its x_old in the window (rows in sweep order, so the north value is
//     read before it is overwritten).  The partner nodes across the two start faces (the
//     other halves of the coupled systems) get their r0 the same way from
//     the halo, redundantly in both boxes.
//  3. Corner and start-face chains: lane 0 solves the corner set (4 x 4, eq 2d:sor4b4, or
//     2 x 2 / 1 x 1); then lane 0 runs the chain of 2 x 2 systems along local row 0 and
//     lane 1 the chain along local column 0 (eq 2d:sor2b2), or the plain recurrence when
//     the face is a physical boundary.
//  4. Wavefront on rows 1..63 x columns 1..63: lane l owns rows 2l+1 and 2l+2 and at step s
//     updates column c = s - l + 1 of both:
//        u_A = fma(a, S, fma(a, W_A, r0_A)),   u_B = fma(a, u_A, fma(a, W_B, r0_B))
//     with W from the lane's registers and S from lane l-1 by shfl.up (lane 0: row 0 in
//     shared memory).  94 steps, in place.
//  5. Write-back: 64 one-row bulk copies (cp.async.bulk) of the box to x_new.
// Elimination order and every fused operation follow the oracle (DESIGN R-7, R-8), so the
// result is bitwise identical to it, independent of CTA schedule and GPU count.
#pragma once
#include <cuda.h>

#include "common.cuh"
#include "tma.cuh"

namespace sw {

namespace p2 {
constexpr int T = 64;       // box edge
constexpr int W = 68;       // window edge
constexpr int WS = W * W;
constexpr int RING = 8;     // b rows in flight in the prologue
constexpr size_t SMEM = sizeof(double) * WS;
}  // namespace p2

struct Sweep2pArgs {
    Geo G;
    int base;
    double omega[4];
    const double *b;     // padded b
    double *xnew;        // padded x_new
    int *flag;
};

__device__ __forceinline__ void prefetch_l2(const void *p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// Gaussian elimination without pivoting (oracle ge_solve, DESIGN R-8).
template <int K>
__device__ __forceinline__ void ge_solve_k(double (&M)[K][K], double (&rhs)[K], double (&u)[K], int *flag) {
    double inv[K];
#pragma unroll
    for (int p = 0; p < K; ++p) {
        const double piv = M[p][p];
        if (!(fabs(piv) >= 1e-14)) atomicOr(flag, 1);
        inv[p] = 1.0 / piv;
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

template <int SX, int SY>
__device__ __forceinline__ void sweep2p_tile(const Sweep2pArgs &A, double *xw, uint64_t *bar, int tx, int ty,
                                             bool cx, bool cy) {
    using namespace p2;
    const Geo &G = A.G;
    const int lane = threadIdx.x;
    const int64_t P0 = G.P0;
    const int x0 = tx * T;                        // padded column of the window origin
    const int64_t y0 = (int64_t)ty * T;           // padded (slab-local) row of the window origin
    constexpr int bits = SX | (SY << 1);
    constexpr int dX = SX ? -1 : 1;               // window step for local +x
    constexpr int dY = SY ? -W : W;               // window step for local +y
    auto WX = [](int c) { return 2 + (SX ? T - 1 - c : c); };
    auto WY = [](int t) { return 2 + (SY ? T - 1 - t : t); };
    auto WI = [&](int c, int t) { return WY(t) * W + WX(c); };
    const double *Bg = A.b;
    auto BG = [&](int wi) { return Bg + (y0 + wi / W) * P0 + (x0 + wi % W); };   // b at window word wi

    const double ap = 4.0 + G.beta;              // a_P = (1 + 1) + (1 + 1) + beta
    const double w_o = A.omega[bits], w_x = A.omega[bits ^ 1], w_y = A.omega[bits ^ 2], w_d = A.omega[bits ^ 3];
    const double al = w_o / ap, al_x = w_x / ap, al_y = w_y / ap, al_d = w_d / ap;
    const double omw = 1.0 - w_o;

    // ---------------------------------------------------------------- 1. stage-in
    const int wc = 2 + 2 * lane;                  // prologue: window columns wc, wc + 1
    auto brow = [&](int t) { return reinterpret_cast<const double2 *>(Bg + (y0 + WY(t)) * P0 + x0 + wc); };
    double2 ring[RING];
#pragma unroll
    for (int k = 0; k < RING; ++k) ring[k] = __ldg(brow(k));
    prefetch_l2(brow(RING + lane), T * sizeof(double));                 // rows RING .. RING+31
    if (lane < T - RING - 32) prefetch_l2(brow(RING + 32 + lane), T * sizeof(double));
    // right-hand sides of the partner nodes
    double bpx[2] = {0.0, 0.0}, bpy[2] = {0.0, 0.0}, bpd = 0.0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int k = h * 32 + lane;
        if (cx) bpx[h] = __ldg(BG(WI(0, k) - dX));
        if (cy) bpy[h] = __ldg(BG(WI(k, 0) - dY));
    }
    const int i00 = WI(0, 0);
    if (cx && cy && lane == 0) bpd = __ldg(BG(i00 - dX - dY));
    mbar_wait(bar, 0);

    // ---------------------------------------------------------------- 2a. partner r0 (halo)
    // A partner across the x face sweeps x the other way and y our way: explicit
    // neighbours (-2, k) and (-1, k+1).  Across the y face: (k+1, -1) and (k, -2).
    double rpx[2], rpy[2], rpd = 0.0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int k = h * 32 + lane;
        const int ix = WI(0, k) - dX, iy = WI(k, 0) - dY;
        rpx[h] = fma(al_x, (bpx[h] + xw[ix - dX]) + xw[ix + dY], (1.0 - w_x) * xw[ix]);
        rpy[h] = fma(al_y, (bpy[h] + xw[iy + dX]) + xw[iy - dY], (1.0 - w_y) * xw[iy]);
    }
    if (lane == 0) {
        const int id = i00 - dX - dY;
        rpd = fma(al_d, (bpd + xw[id - dX]) + xw[id - dY], (1.0 - w_d) * xw[id]);
    }
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int k = h * 32 + lane;
        if (cx) xw[WI(0, k) - dX] = rpx[h];
        if (cy) xw[WI(k, 0) - dY] = rpy[h];
    }
    if (cx && cy && lane == 0) xw[i00 - dX - dY] = rpd;

    // ---------------------------------------------------------------- 2b. own r0 (rows in sweep order)
#pragma unroll 1
    for (int t0 = 0; t0 < T; t0 += RING) {
#pragma unroll
        for (int k = 0; k < RING; ++k) {
            const int t = t0 + k;
            const int i = WY(t) * W + wc;
            const double2 own = *reinterpret_cast<const double2 *>(xw + i);
            const double2 nb = *reinterpret_cast<const double2 *>(xw + i + dY);
            double e0, e1;                             // explicit (local +x) neighbours
            if constexpr (SX) {
                const double up = __shfl_up_sync(0xffffffffu, own.y, 1);
                e0 = (lane == 0) ? xw[i - 1] : up;
                e1 = own.x;
            } else {
                const double dn = __shfl_down_sync(0xffffffffu, own.x, 1);
                e0 = own.y;
                e1 = (lane == 31) ? xw[i + 2] : dn;
            }
            const double2 bb = ring[k];
            const double r00 = fma(al, (bb.x + e0) + nb.x, omw * own.x);
            const double r01 = fma(al, (bb.y + e1) + nb.y, omw * own.y);
            *reinterpret_cast<double2 *>(xw + i) = make_double2(r00, r01);
            if (t + RING < T) ring[k] = __ldg(brow(t + RING));
        }
    }
    __syncwarp();

    // ---------------------------------------------------------------- 3. corner and chains
    if (lane == 0) {
        if (cx && cy) {
            // members in ascending global index: (lo y, lo x), (lo y, hi x), (hi y, lo x), (hi y, hi x)
            constexpr int xlo_p = (SX == 0), ylo_p = (SY == 0);
            double M[4][4], rhs[4], uu[4];
            int idx[4];
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                const int isx = (m & 1) ? !xlo_p : xlo_p;       // member on the partner side of x
                const int isy = (m & 2) ? !ylo_p : ylo_p;
                idx[m] = i00 - (isx ? dX : 0) - (isy ? dY : 0);
                const double a = (isx && isy) ? al_d : (isx ? al_x : (isy ? al_y : al));
#pragma unroll
                for (int q = 0; q < 4; ++q) M[m][q] = (m == q) ? 1.0 : 0.0;
                rhs[m] = xw[idx[m]];
                M[m][m ^ 1] = -a;
                M[m][m ^ 2] = -a;
            }
            ge_solve_k<4>(M, rhs, uu, A.flag);
#pragma unroll
            for (int m = 0; m < 4; ++m) xw[idx[m]] = uu[m];
        } else if (cx || cy) {
            const int ip = cx ? i00 - dX : i00 - dY;
            const double ap_ = cx ? al_x : al_y;
            const bool pfirst = cx ? (SX == 0) : (SY == 0);
            double M[2][2], rhs[2], uu[2];
            M[0][0] = M[1][1] = 1.0;
            rhs[0] = pfirst ? xw[ip] : xw[i00];
            rhs[1] = pfirst ? xw[i00] : xw[ip];
            M[0][1] = -(pfirst ? ap_ : al);
            M[1][0] = -(pfirst ? al : ap_);
            ge_solve_k<2>(M, rhs, uu, A.flag);
            xw[i00] = pfirst ? uu[1] : uu[0];
            xw[ip] = pfirst ? uu[0] : uu[1];
        }
        // (no coupling: u(0,0) = r0, already in place)
    }
    __syncwarp();
    if (lane < 2) {
        // lane 0: chain along local row 0 (pairs across the y start face)
        // lane 1: chain along local column 0 (pairs across the x start face)
        const int step = lane ? dY : dX;
        const int perp = lane ? dX : dY;
        const bool coupled = lane ? cx : cy;
        const bool pfirst = lane ? (SX == 0) : (SY == 0);
        const double alp = lane ? al_x : al_y;
        // member a = lower global index; row a: u_a - m_ab u_b = r_a
        const double mab = pfirst ? alp : al, mba = pfirst ? al : alp;
        const double M11 = fma(mba, -mab, 1.0);
        if (coupled && !(fabs(M11) >= 1e-14)) atomicOr(A.flag, 1);
        const double inv1 = 1.0 / M11;
        int io = i00;
        double po = xw[io], pp = coupled ? xw[io - perp] : 0.0;
#pragma unroll 4
        for (int k = 1; k < T; ++k) {
            io += step;
            const double ro = fma(al, po, xw[io]);
            if (coupled) {
                const double rp = fma(alp, pp, xw[io - perp]);
                const double ra = pfirst ? rp : ro, rb = pfirst ? ro : rp;
                const double ub = fma(mba, ra, rb) * inv1;
                const double ua = fma(mab, ub, ra) * 1.0;
                po = pfirst ? ub : ua;
                pp = pfirst ? ua : ub;
                xw[io - perp] = pp;
            } else {
                po = ro;
            }
            xw[io] = po;
        }
    }
    __syncwarp();

    // ---------------------------------------------------------------- 4. wavefront
    {
        const int rA = 2 * lane + 1;                       // rows A = 2l+1, B = 2l+2 (lane 31: B = 64, halo)
        double *pA = xw + WI(1, rA);                       // node (c, A) at pA + (c-1) dX
        double WA = pA[-dX];                               // u(0, A), u(0, B) from the column chain
        double WB = pA[dY - dX];
        double uB = 0.0;
        auto stepf = [&](int s, bool pred) {
            const int c = s - lane + 1;
            const bool act = !pred || (c >= 1 && c <= T - 1);
            double *p = pA + (c - 1) * dX;
            const double r0A = p[0], r0B = p[dY];
            const double row0 = p[-(rA)*dY];               // u(c, 0): only lane 0 uses it
            const double sh = __shfl_up_sync(0xffffffffu, uB, 1);
            const double S = (lane == 0) ? row0 : sh;
            const double uA = fma(al, S, fma(al, WA, r0A));
            const double nB = fma(al, uA, fma(al, WB, r0B));
            if (act) {
                p[0] = uA;
                if (lane < 31) p[dY] = nB;
                WA = uA;
                WB = nB;
                uB = nB;
            }
        };
        // ramp-up: lane l joins at step l; steady: all 32 lanes; ramp-down: lane l leaves after step l + 62
#pragma unroll 2
        for (int s = 0; s < 31; ++s) stepf(s, true);
#pragma unroll 4
        for (int s = 31; s < 63; ++s) stepf(s, false);
#pragma unroll 2
        for (int s = 63; s < 94; ++s) stepf(s, true);
    }

    // ---------------------------------------------------------------- 5. write-back
    fence_proxy_async_smem();
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int r = h * 32 + lane;                       // window row 2 + r
        double *dst = A.xnew + (y0 + r + 2) * P0 + (x0 + 2);
        bulk_store(dst, xw + (r + 2) * W + 2, T * sizeof(double));
    }
    bulk_commit();
    bulk_wait_read0();
}

__global__ void __launch_bounds__(32, 6) k_sweep2p(const __grid_constant__ CUtensorMap tmx, Sweep2pArgs A) {
    extern __shared__ __align__(128) double xw[];
    __shared__ uint64_t bar;
    const Geo &G = A.G;
    const int lane = threadIdx.x;
    const int tx = blockIdx.x % G.nt[0];
    const int ty = blockIdx.x / G.nt[0];
    const int64_t R0 = tx, R1 = ty + G.toff[1];
    const int sx = ((A.base >> 0) & 1) ^ (int)(R0 & 1);
    const int sy = ((A.base >> 1) & 1) ^ (int)(R1 & 1);
    const bool cx = sx ? (R0 < G.ntg[0] - 1) : (R0 > 0);
    const bool cy = sy ? (R1 < G.ntg[1] - 1) : (R1 > 0);
    if (lane == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
        mbar_expect_tx(&bar, (uint32_t)p2::SMEM);
        tma_load_2d(xw, &tmx, tx * p2::T, ty * p2::T, &bar);
    }
    __syncwarp();
    switch (sx | (sy << 1)) {
        case 0: sweep2p_tile<0, 0>(A, xw, &bar, tx, ty, cx, cy); break;
        case 1: sweep2p_tile<1, 0>(A, xw, &bar, tx, ty, cx, cy); break;
        case 2: sweep2p_tile<0, 1>(A, xw, &bar, tx, ty, cx, cy); break;
        default: sweep2p_tile<1, 1>(A, xw, &bar, tx, ty, cx, cy); break;
    }
}

inline cudaError_t launch_sweep2p(const CUtensorMap &tmx, const Geo &G, int base, const double *w8, const double *b,
                                  double *xn, int *flag, cudaStream_t s) {
    Sweep2pArgs A;
    A.G = G;
    A.base = base;
    for (int i = 0; i < 4; ++i) A.omega[i] = w8[i];
    A.b = b;
    A.xnew = xn;
    A.flag = flag;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_sweep2p, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p2::SMEM);
        cudaFuncSetAttribute(k_sweep2p, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        attr = true;
    }
    const unsigned tiles = (unsigned)((int64_t)G.nt[0] * G.nt[1]);
    k_sweep2p<<<tiles, 32, p2::SMEM, s>>>(tmx, A);
    return cudaGetLastError();
}

}  // namespace sw
