// sweep2p.cuh -- 2D decomposed SOR sweep, constant coefficients (Poisson), 64 x 64 boxes,
// sm_100a (sweep2v.cuh is the variable-coefficient counterpart).
//
// One CTA = two warps = one box.  Six CTAs fit on an SM (36 KB of shared
// memory each), so 12 warps share the latency of the staged loads.  Per box:
//  1. Stage-in: one TMA load of the 68 x 68 window of x_old (box + 2-node halo,
//     PAPER:828-833) into shared memory; the 64 x 64 b tile is prefetched into L2 by a TMA
//     tensor prefetch and read back coalesced through a register ring.
//  2. Explicit parts (data parallel, coalesced): every owned node's
//        r0 = fma(w/a_P, (b + u_E) + u_N, (1-w) u)         (DESIGN R-7)
//     is written over its x_old in the window (rows in sweep order, so the north value is
//     read before it is overwritten).  The partner nodes across the two start faces (the
//     other halves of the coupled systems) get their r0 the same way from
//     the halo, redundantly in both boxes.
//  3. Corner and start-face chains: lane 0 solves the corner set (4 x 4, eq 2d:sor4b4, or
//     2 x 2 / 1 x 1); then lane 0 runs the chain of 2 x 2 systems along local row 0 and
//     lane 1 the chain along local column 0 (eq 2d:sor2b2), or the plain recurrence when
//     the face is a physical boundary, with one branch-free body for all cases.
//  4. Wavefront on rows 1..63 x columns 1..63: lane l owns rows 2l+1 and 2l+2 and at step s
//     updates column c = s - l + 1 of both:
//        u_A = fma(a, S, fma(a, W_A, r0_A)),   u_B = fma(a, u_A, fma(a, W_B, r0_B))
//     with W from the lane's registers and S from lane l-1 by shfl.up (lane 0: row 0 in
//     shared memory).  94 steps, in place, branch-free (idle lanes of the ramps only
//     predicate their stores).
//  5. Write-back: coalesced 16-byte streaming stores of the 64 rows to x_new (per-lane bulk
//     copies would need uniform operands and compile to a 32-way waterfall loop).
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

__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap *map, int c0, int c1) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(map), "r"(c0), "r"(c1)
                 : "memory");
}

// Branch-free building blocks for the wavefront (the compiler otherwise turns guarded stores
// and selects into divergent branches with reconvergence barriers around every shuffle).
__device__ __forceinline__ void st_shared_if(double *addr, double v, bool pred) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %2, 0;\n @p st.shared.f64 [%0], %1;\n}\n" ::"r"(smem_u32(addr)), "d"(v),
        "r"((int)pred)
        : "memory");
}
__device__ __forceinline__ double sel_f64(bool pred, double a, double b) {
    double r;
    asm("{\n .reg .pred p;\n setp.ne.b32 p, %1, 0;\n selp.f64 %0, %2, %3, p;\n}\n" : "=d"(r) : "r"((int)pred), "d"(a), "d"(b));
    return r;
}
__device__ __forceinline__ double shfl_up1_f64(double v) {   // full warp, converged by construction
    int lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "d"(v));
    asm volatile("shfl.sync.up.b32 %0, %0, 1, 0, 0xffffffff;" : "+r"(lo));
    asm volatile("shfl.sync.up.b32 %0, %0, 1, 0, 0xffffffff;" : "+r"(hi));
    double r;
    asm("mov.b64 %0, {%1, %2};" : "=d"(r) : "r"(lo), "r"(hi));
    return r;
}

// Gaussian elimination without pivoting (oracle ge_solve, DESIGN R-8).
template <int K>
__device__ __forceinline__ void ge_solve_k(double (&M)[K][K], double (&rhs)[K], double (&u)[K], int *flag) {
    double inv[K];
#pragma unroll
    for (int p = 0; p < K; ++p) {
        const double piv = M[p][p];
        if (!(fabs(piv) >= 1e-14)) atomicOr(flag, 1);
        inv[p] = div_rn(1.0, piv);          // = 1.0 / piv (IEEE), without the slow-path call
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
    const int warp = threadIdx.x >> 5;            // two warps per box
    const int lane = threadIdx.x & 31;
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
    const int i00 = WI(0, 0);
    SW_TMARK(t_start);

    // ---------------------------------------------------------------- 1. stage-in
    // Warp w computes local rows 32w .. 32w+31 of the prologue; its b rows stream through a
    // register ring (the whole b tile was prefetched into L2 with the TMA load).
    const int wc = 2 + 2 * lane;                  // prologue: window columns wc, wc + 1
    const int t_first = warp * (T / 2);
    const int64_t bstep = (SY ? -P0 : P0) / 2;    // one local row of b, in double2 (P0 % 8 == 0)
    const double2 *bp = reinterpret_cast<const double2 *>(Bg + (y0 + WY(t_first)) * P0 + x0 + wc);
    double2 ring[RING];
#pragma unroll
    for (int k = 0; k < RING; ++k) ring[k] = __ldg(bp + k * bstep);
    bp += RING * bstep;
    // right-hand sides of the partner nodes: warp 0 the y-face row, warp 1 the x-face column
    // (and the diagonal corner partner)
    double bp2[2] = {0.0, 0.0}, bpd = 0.0;
    const bool cpl = warp ? cx : cy;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int k = h * 32 + lane;
        if (cpl) bp2[h] = __ldg(BG(warp ? WI(0, k) - dX : WI(k, 0) - dY));
    }
    if (cx && cy && warp == 1 && lane == 0) bpd = __ldg(BG(i00 - dX - dY));
    mbar_wait(bar, 0);
    SW_TMARK(t_staged);

    // ---------------------------------------------------------------- 2a. partner r0 (halo)
    // A partner across the x face sweeps x the other way and y our way: explicit
    // neighbours (-2, k) and (-1, k+1).  Across the y face: (k+1, -1) and (k, -2).
    {
        const double alp = warp ? al_x : al_y, omp = 1.0 - (warp ? w_x : w_y);
        const int ex = warp ? -dX : dX, ey = warp ? dY : -dY;   // explicit neighbour offsets
        double rp[2], rpd = 0.0;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int k = h * 32 + lane;
            const int ip = warp ? WI(0, k) - dX : WI(k, 0) - dY;
            rp[h] = fma(alp, (bp2[h] + xw[ip + ex]) + xw[ip + ey], omp * xw[ip]);
        }
        const int id = i00 - dX - dY;
        if (warp == 1 && lane == 0) rpd = fma(al_d, (bpd + xw[id - dX]) + xw[id - dY], (1.0 - w_d) * xw[id]);
        // warp 0 keeps the old values of row 32 (the north neighbours of its last row)
        double2 save = make_double2(0.0, 0.0);
        if (warp == 0) save = *reinterpret_cast<const double2 *>(xw + WY(T / 2) * W + wc);
        __syncthreads();
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int k = h * 32 + lane;
            if (cpl) xw[warp ? WI(0, k) - dX : WI(k, 0) - dY] = rp[h];
        }
        if (cx && cy && warp == 1 && lane == 0) xw[id] = rpd;

        // ------------------------------------------------------------ 2b. own r0 (rows in sweep order)
        double *px = xw + WY(t_first) * W + wc;
        double2 cur = *reinterpret_cast<const double2 *>(px);
        auto row = [&](double2 bb, bool last) {
            const double2 nb = (last && warp == 0) ? save : *reinterpret_cast<const double2 *>(px + dY);
            double e0, e1;                                                    // explicit (local +x) neighbours
            if constexpr (SX) {
                const double up = __shfl_up_sync(0xffffffffu, cur.y, 1);
                e0 = (lane == 0) ? px[-1] : up;
                e1 = cur.x;
            } else {
                const double dn = __shfl_down_sync(0xffffffffu, cur.x, 1);
                e0 = cur.y;
                e1 = (lane == 31) ? px[2] : dn;
            }
            const double r00 = fma(al, (bb.x + e0) + nb.x, omw * cur.x);
            const double r01 = fma(al, (bb.y + e1) + nb.y, omw * cur.y);
            *reinterpret_cast<double2 *>(px) = make_double2(r00, r01);
            cur = nb;
            px += dY;
        };
#pragma unroll 1
        for (int t0 = 0; t0 < T / 2 - RING; t0 += RING) {
#pragma unroll
            for (int k = 0; k < RING; ++k) {
                row(ring[k], false);
                ring[k] = __ldg(bp);
                bp += bstep;
            }
        }
#pragma unroll
        for (int k = 0; k < RING; ++k) row(ring[k], k == RING - 1);
    }
    __syncthreads();

    SW_TMARK(t_prologue);
    // ---------------------------------------------------------------- 3. corner and chains (warp 1)
    SW_TMARK(t_c0);
    if (warp == 1 && lane == 0) {
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
    if (warp == 1 && lane < 2) {
        // lane 0: chain along local row 0 (pairs across the y start face)
        // lane 1: chain along local column 0 (pairs across the x start face)
        // Kept in member order: a = lower global index, row a: u_a - m_ab u_b = r_a (oracle
        // ge_solve: u_b = fma(m_ba, r_a, r_b) / (1 - m_ba m_ab), u_a = fma(m_ab, u_b, r_a)).
        // An uncoupled face (physical boundary) runs the same code with b = own node, a = the
        // zero ghost node and m_ab = m_ba = 0, which leaves u_b = fma(al, W, r0) exactly.
        const int step = lane ? dY : dX;
        const int perp = lane ? dX : dY;
        const bool coupled = lane ? cx : cy;
        const bool pfirst = lane ? (SX == 0) : (SY == 0);
        const double alp = lane ? al_x : al_y;
        const bool a_is_p = pfirst || !coupled;
        int ia = a_is_p ? i00 - perp : i00;
        int ib = a_is_p ? i00 : i00 - perp;
        const double ma = coupled ? (pfirst ? alp : al) : 0.0;
        const double mb = pfirst || !coupled ? al : alp;
        const double mab = coupled ? ma : 0.0, mba = coupled ? mb : 0.0;
        const double M11 = fma(mba, -mab, 1.0);
        if (coupled && !(fabs(M11) >= 1e-14)) atomicOr(A.flag, 1);
        const double inv1 = coupled ? 1.0 / M11 : 1.0;
        double pa = xw[ia], pb = xw[ib];
        // loads of step k+1 are issued before the stores of step k (they never alias, but the
        // compiler cannot prove it for a run-time stride)
        double na = xw[ia + step], nb = xw[ib + step];
#pragma unroll 4
        for (int k = 1; k < T; ++k) {
            ia += step;
            ib += step;
            const double r0a = na, r0b = nb;
            na = xw[ia + step];
            nb = xw[ib + step];
            const double ra = fma(ma, pa, r0a);
            const double rb = fma(mb, pb, r0b);
            pb = fma(mba, ra, rb) * inv1;
            pa = fma(mab, pb, ra);
            xw[ia] = pa;
            xw[ib] = pb;
        }
    }
    __syncwarp();
    SW_TMARK(t_c1);
    SW_TADDT(6, t_c0, t_c1, 32);

    // ---------------------------------------------------------------- 4. wavefront (warp 0)
    __syncthreads();
    SW_TMARK(t_chains);
    SW_TMARK(t_w0);
    if (warp == 0) {
        // Lane l owns rows A = 2l+1, B = 2l+2 (lane 31: B = 64, halo, never stored) and at step
        // s updates column c = s - SKEW l + 1 of both.  SKEW = 2 would give the shuffle carrying
        // u_B of lane l-1 (needed as S by lane l) a whole step to arrive, at the price of 31
        // more steps; measured, SKEW = 1 is faster.
#ifndef SW_SKEW
#define SW_SKEW 1
#endif
        constexpr int SKEW = SW_SKEW, NSTEP = (T - 1) + SKEW * 31;
        const int rA = 2 * lane + 1;
        double *pA = xw + WI(1, rA);                       // node (c, A) at pA + (c-1) dX
        double WA = pA[-dX];                               // u(0, A), u(0, B) from the column chain
        double WB = pA[dY - dX];
        double uBp = 0.0, shv = 0.0;
        // values of the current step, loaded during the previous one (before its stores: the
        // addresses never alias, but the row-0 offset is lane dependent and the compiler
        // would otherwise order every load after the previous step's stores)
        double *p = pA + (-SKEW * lane) * dX;             // step 0: c = 1 - SKEW l
        double nr0A = p[0], nr0B = p[dY], nrow0 = p[-(rA)*dY];
        // RAMP: 1 = lanes join (lane l is idle before step SKEW l and keeps W = u(0, .)),
        // 2 = lanes leave (lane l is done after step SKEW l + 62).  Branch-free: idle lanes
        // only suppress their stores and, while joining, their W updates.  (u_B needs no
        // guard: lane l+1 uses it only when lane l was busy.)
        auto stepf = [&](int s, int RAMP) {
            const int c = s - SKEW * lane + 1;
            const bool act = RAMP == 1 ? c >= 1 : c <= T - 1;
            const double r0A = nr0A, r0B = nr0B, row0 = nrow0;  // u(c, 0): only lane 0 uses row0
            double *q = p + dX;
            nr0A = q[0];
            nr0B = q[dY];
            nrow0 = q[-(rA)*dY];
            double S;                                           // u_B of lane l-1 at column c
            if constexpr (SKEW == 1) {                          // computed in the previous step
                S = sel_f64(lane == 0, row0, shfl_up1_f64(uBp));
            } else {                                            // two steps ago: shuffled last step
                S = sel_f64(lane == 0, row0, shv);
                shv = shfl_up1_f64(uBp);
            }
            const double uA = fma(al, S, fma(al, WA, r0A));
            const double nB = fma(al, uA, fma(al, WB, r0B));
            st_shared_if(p, uA, act);
            st_shared_if(p + dY, nB, act && lane < 31);
            if (RAMP == 1) {
                WA = sel_f64(act, uA, WA);
                WB = sel_f64(act, nB, WB);
            } else {
                WA = uA;
                WB = nB;
            }
            uBp = nB;
            p = q;
        };
#pragma unroll 4
        for (int s = 0; s < SKEW * 31; ++s) stepf(s, 1);
#pragma unroll 4
        for (int s = SKEW * 31; s < NSTEP; ++s) stepf(s, 2);
        SW_TMARK(t_w1);
        SW_TADDT(7, t_w0, t_w1, 0);
    }

    // ---------------------------------------------------------------- 5. write-back (32 rows per warp)
    __syncthreads();
    SW_TMARK(t_wave);
    {
        const int r0 = 2 + warp * (T / 2);
        const double *src = xw + r0 * W + wc;
        double2 *dst = reinterpret_cast<double2 *>(A.xnew + (y0 + r0) * P0 + x0 + wc);
#pragma unroll 8
        for (int r = 0; r < T / 2; ++r) {
            const double2 v = *reinterpret_cast<const double2 *>(src + r * W);
            __stcs(dst + r * (P0 / 2), v);
        }
    }
    SW_TMARK(t_end);
    SW_TADD(0, t_start, t_staged);
    SW_TADD(1, t_staged, t_prologue);
    SW_TADD(2, t_prologue, t_chains);
    SW_TADD(3, t_chains, t_wave);
    SW_TADD(4, t_wave, t_end);
    SW_TADD(5, 0, 1);
}

__global__ void __launch_bounds__(64, 6)
    k_sweep2p(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmb, Sweep2pArgs A) {
    extern __shared__ __align__(128) double xw[];
    __shared__ uint64_t bar;
    SW_JITTER_POINT();
    const Geo &G = A.G;
    const int tid = threadIdx.x;
    const int tx = blockIdx.x % G.nt[0];
    const int ty = blockIdx.x / G.nt[0];
    const int64_t R0 = tx, R1 = ty + G.toff[1];
    const int sx = ((A.base >> 0) & 1) ^ (int)(R0 & 1);
    const int sy = ((A.base >> 1) & 1) ^ (int)(R1 & 1);
    const bool cx = sx ? (R0 < G.ntg[0] - 1) : (R0 > 0);
    const bool cy = sy ? (R1 < G.ntg[1] - 1) : (R1 > 0);
    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
        mbar_expect_tx(&bar, (uint32_t)p2::SMEM);
        tma_load_2d(xw, &tmx, tx * p2::T, ty * p2::T, &bar);
        tma_prefetch_2d(&tmb, tx * p2::T + 2, ty * p2::T + 2);      // b tile into L2
    }
    __syncthreads();
    switch (sx | (sy << 1)) {
        case 0: sweep2p_tile<0, 0>(A, xw, &bar, tx, ty, cx, cy); break;
        case 1: sweep2p_tile<1, 0>(A, xw, &bar, tx, ty, cx, cy); break;
        case 2: sweep2p_tile<0, 1>(A, xw, &bar, tx, ty, cx, cy); break;
        default: sweep2p_tile<1, 1>(A, xw, &bar, tx, ty, cx, cy); break;
    }
}

inline cudaError_t launch_sweep2p(const CUtensorMap &tmx, const CUtensorMap &tmb, const Geo &G, int base, const double *w8, const double *b,
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
    k_sweep2p<<<tiles, 64, p2::SMEM, s>>>(tmx, tmb, A);
    return cudaGetLastError();
}

}  // namespace sw
