// sweep2v.cuh -- 2D decomposed SOR sweep, variable coefficients (face arrays F_x, F_y),
// 64 x 64 boxes, sm_100a.  Same structure as the constant-coefficient kernel (sweep2p.cuh);
// what differs is that every node carries its own couplings:
//
//  a_P = ((F_x- + F_x+) + (F_y- + F_y+)) + beta,  alpha = w / a_P,
//  r0  = fma(alpha, fma(c_N, u_N, fma(c_E, u_E, b)), (1 - w) u),
//  m_W = alpha c_W,  m_S = alpha c_S,   u = fma(m_S, S, fma(m_W, W, r0))     (DESIGN R-7)
//
// One CTA = eight warps = one box; 105 KB of shared memory (x window with r0 in place, m_W and
// m_S per node, the partner couplings of the start-face chains), two CTAs per SM.
//  1. Stage-in: TMA load of the 68 x 68 x_old window; TMA tensor prefetches of the b, F_x
//     and F_y tiles into L2; each warp streams its rows of b / F_x / F_y through a register ring.
//  2. Partners (warps 0, 1): r0 and couplings of the y-face row, the x-face column and the
//     diagonal corner partner; explicit parts of the own nodes (all warps, 8 rows each, in
//     sweep order), one IEEE division per node.
//  3. Corner set and the two start-face chains (warp 1, lanes 0 and 1).
//  4. Wavefront (warp 0): lane l owns rows 2l+1, 2l+2; 94 branch-free steps.
//  5. Coalesced write-back (all warps).
// Bitwise identical to the oracle (same operations in the same order).
#pragma once
#include <cuda.h>

#include "common.cuh"
#include "sweep2p.cuh"
#include "tma.cuh"

namespace sw {

namespace v2 {
constexpr int T = 64, W = 68, WS = W * W;
#ifndef SW_V2_NW
#define SW_V2_NW 8
#endif
constexpr int NW = SW_V2_NW;            // warps per box (8: the prologue streams 8 rows per warp)
constexpr int ROWS = T / NW;            // prologue rows per warp
#ifndef SW_V2_RING
#define SW_V2_RING 2
#endif
constexpr int RING = SW_V2_RING;        // rows in flight per warp
constexpr int NCOEF = T * T;            // m_W / m_S arrays, pitch 64 (window column order)
constexpr int NCH = 6 * T + 4;          // chain partner couplings, chain pivots, diagonal couplings, 0, 1
constexpr size_t SMEM = sizeof(double) * (WS + 2 * NCOEF + NCH);
}  // namespace v2

// MODE_SOR: one decomposed SOR sweep (window = x_old, aux = b).
// MODE_TRI: one block-triangular solve (D/alpha + A_I) out = r (the ILU / SSOR factors,
//   SURVEY §8(a) a11-a12): window = src, r0 = alpha src (rscale) or coef src, alpha = 1/D~ from
//   aux (invd_mode, ILU) or omega / a_P (SSOR); couple = 0 drops the start-face coupling (the
//   first phase of the transposed solve, run at the reversed corner).
enum { MODE_SOR = 0, MODE_TRI = 1 };

// Look-ahead (SW_V2_AHEAD boxes, 0 = off): once its own prologue is done, a box asks the L2 for the
// tiles of the box that will take its place on the SM (x window, aux, F_x, F_y), so that box's
// stage-in and prologue find their lines in L2 instead of waiting on HBM.
#ifndef SW_V2_AHEAD
#define SW_V2_AHEAD 222
#endif
struct Ahead2v {
    const CUtensorMap *x, *b, *fx, *fy;
    int tx, ty;        // tile coordinates of the box looked ahead to (tx < 0: none)
};

struct Sweep2vArgs {
    Geo G;
    int base;
    double omega[4];
    const double *b, *fx, *fy;   // padded aux (b or 1/D~), F_x, F_y
    double *xnew;
    int *flag;
    double coef;
    int invd_mode, rscale, couple;
};

// Shared-memory store that the compiler does not treat as a memory clobber: used for the
// coupling arrays, which no load of the same phase reads (the explicit-part loads of later
// rows would otherwise be ordered after every coupling store).
__device__ __forceinline__ void st_shared_v2_noalias(double *addr, double a, double b) {
    asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(smem_u32(addr)), "d"(a), "d"(b));
}

template <int MODE, bool FACES, int SX, int SY>
__device__ __forceinline__ void sweep2v_tile(const Sweep2vArgs &A, double *sm, uint64_t *bar, int tx, int ty, bool cx,
                                             bool cy, const Ahead2v &AH) {
    constexpr bool SOR = (MODE == MODE_SOR);
    const bool invd = !SOR && A.invd_mode;      // alpha = 1/D~ from the aux array (ILU)
    const bool load_aux = SOR || invd;
    using namespace v2;
    double *xw = sm;                       // x window; r0 and results in place
    double *cW = xw + WS;                  // m_W per own node, index (wr-2)*64 + (wc-2)
    double *cS = cW + NCOEF;               // m_S
    double *ych_c = cS + NCOEF;            // y-face partner (k,-1): coupling to (k-1,-1)
    double *ych_p = ych_c + T;             //                        coupling to own (k,0)
    double *xch_c = ych_p + T;             // x-face partner (-1,k): coupling to (-1,k-1)
    double *xch_p = xch_c + T;             //                        coupling to own (0,k)
    double *inv_y = xch_p + T;             // 1 / (1 - m_own m_partner) of the y-face pairs (k,0),(k,-1)
    double *inv_x = inv_y + T;             //                              x-face pairs (0,k),(-1,k)
    double *dg = inv_x + T;                // [0] diagonal -> (0,-1), [1] diagonal -> (-1,0), [2] = 0, [3] = 1

    const Geo &G = A.G;
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t P0 = G.P0;
    const int x0 = tx * T;
    const int64_t y0 = (int64_t)ty * T;
    constexpr int bits = SX | (SY << 1);
    constexpr int dX = SX ? -1 : 1;
    constexpr int dY = SY ? -W : W;
    constexpr int dYc = SY ? -T : T;       // local +y in the coefficient arrays
    auto WX = [](int c) { return 2 + (SX ? T - 1 - c : c); };
    auto WY = [](int t) { return 2 + (SY ? T - 1 - t : t); };
    auto WI = [&](int c, int t) { return WY(t) * W + WX(c); };
    auto CI = [&](int c, int t) { return (WY(t) - 2) * T + (WX(c) - 2); };
    auto PI = [&](int wi) { return (y0 + wi / W) * P0 + (x0 + wi % W); };   // padded index of window word
    const double *Bg = A.b, *Fx = A.fx, *Fy = A.fy;
    const double beta = G.beta;
    const double w_o = A.omega[bits], w_x = A.omega[bits ^ 1], w_y = A.omega[bits ^ 2], w_d = A.omega[bits ^ 3];
    const double omw = 1.0 - w_o;
    const int i00 = WI(0, 0), c00 = CI(0, 0);
    SW_TMARK(t_start);

    // ---------------------------------------------------------------- 1. stage-in
    const int wc = 2 + 2 * lane;
    const int t_first = warp * ROWS;
    const int64_t rstep = SY ? -P0 : P0;                       // one local row in the padded arrays
    const int64_t g_first = (y0 + WY(t_first)) * P0 + x0 + wc;  // padded index of (wc, row t_first)
    const double *pb = Bg + g_first, *pfx = Fx + g_first;
    const double *pfy = Fy + g_first + (SY ? 0 : P0);          // the F_y row each local row brings in
    double2 rb[RING], rfx[RING], rfy[RING];
    double rfe[RING];
#pragma unroll
    for (int k = 0; k < RING; ++k) {
        rb[k] = load_aux ? __ldg(reinterpret_cast<const double2 *>(pb + k * rstep)) : make_double2(0.0, 0.0);
        if constexpr (FACES) {
            rfx[k] = __ldg(reinterpret_cast<const double2 *>(pfx + k * rstep));
            rfe[k] = (lane == 31) ? __ldg(pfx + k * rstep + 2) : 0.0;
            rfy[k] = __ldg(reinterpret_cast<const double2 *>(pfy + k * rstep));
        } else {
            rfx[k] = rfy[k] = make_double2(1.0, 1.0);
            rfe[k] = 1.0;
        }
    }
    // F_y row carried in from the row before the first one
    double2 fcarry = make_double2(1.0, 1.0);
    if constexpr (FACES) fcarry = __ldg(reinterpret_cast<const double2 *>(Fy + g_first + (SY ? P0 : 0)));
    pb += RING * rstep;
    pfx += RING * rstep;
    pfy += RING * rstep;
    mbar_wait(bar, 0);
    SW_TMARK(t_staged);

    // ---------------------------------------------------------------- 2a. partners (warps 0, 1)
    // faces of the node at window word i, global orientation: xl = F_x(i), xh = F_x(i+1),
    // yl = F_y(i), yh = F_y(i + row)
    double rp[2] = {0.0, 0.0}, mc[2] = {0.0, 0.0}, mp[2] = {0.0, 0.0}, rpd = 0.0, dmx = 0.0, dmy = 0.0;
    const bool cpl = warp == 1 ? cx : cy;
    if (warp < 2) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int k = h * 32 + lane;
            const int ip = warp ? WI(0, k) - dX : WI(k, 0) - dY;
            const int64_t g = PI(ip);
            double xl = 1.0, xh = 1.0, yl = 1.0, yh = 1.0;
            if constexpr (FACES) {
                xl = __ldg(Fx + g); xh = __ldg(Fx + g + 1); yl = __ldg(Fy + g); yh = __ldg(Fy + g + P0);
            }
            const double bv = load_aux ? __ldg(Bg + g) : 0.0;
            const double ap = ((xl + xh) + (yl + yh)) + beta;
            if (warp == 0) {        // y-face partner: x as ours, y flipped
                const double al = invd ? bv : div_rn(w_y, ap);
                if constexpr (SOR) {
                    const double e = fma(SY ? yh : yl, xw[ip - dY], fma(SX ? xl : xh, xw[ip + dX], bv));
                    rp[h] = fma(al, e, (1.0 - w_y) * xw[ip]);
                } else {
                    rp[h] = A.rscale ? al * xw[ip] : A.coef * xw[ip];
                }
                mc[h] = al * (SX ? xh : xl);
                mp[h] = al * (SY ? yl : yh);
            } else {                // x-face partner: x flipped, y as ours
                const double al = invd ? bv : div_rn(w_x, ap);
                if constexpr (SOR) {
                    const double e = fma(SY ? yl : yh, xw[ip + dY], fma(SX ? xh : xl, xw[ip - dX], bv));
                    rp[h] = fma(al, e, (1.0 - w_x) * xw[ip]);
                } else {
                    rp[h] = A.rscale ? al * xw[ip] : A.coef * xw[ip];
                }
                mc[h] = al * (SY ? yh : yl);
                mp[h] = al * (SX ? xl : xh);
            }
        }
        if (warp == 1 && lane == 0) {   // diagonal partner: both flipped
            const int id = i00 - dX - dY;
            const int64_t g = PI(id);
            double xl = 1.0, xh = 1.0, yl = 1.0, yh = 1.0;
            if constexpr (FACES) {
                xl = __ldg(Fx + g); xh = __ldg(Fx + g + 1); yl = __ldg(Fy + g); yh = __ldg(Fy + g + P0);
            }
            const double bv = load_aux ? __ldg(Bg + g) : 0.0;
            const double ap = ((xl + xh) + (yl + yh)) + beta;
            const double al = invd ? bv : div_rn(w_d, ap);
            if constexpr (SOR) {
                const double e = fma(SY ? yh : yl, xw[id - dY], fma(SX ? xh : xl, xw[id - dX], bv));
                rpd = fma(al, e, (1.0 - w_d) * xw[id]);
            } else {
                rpd = A.rscale ? al * xw[id] : A.coef * xw[id];
            }
            dmx = al * (SX ? xl : xh);
            dmy = al * (SY ? yl : yh);
        }
    }
    // each warp keeps the old values of the row after its last one (north of its last row)
    double2 save = make_double2(0.0, 0.0);
    if (SOR && warp < NW - 1) save = *reinterpret_cast<const double2 *>(xw + WY(t_first + ROWS) * W + wc);
    __syncthreads();
    if (warp < 2) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int k = h * 32 + lane;
            if (cpl) xw[warp ? WI(0, k) - dX : WI(k, 0) - dY] = rp[h];
            (warp ? xch_c : ych_c)[k] = mc[h];
            (warp ? xch_p : ych_p)[k] = mp[h];
        }
        if (warp == 1 && lane == 0) {
            if (cx && cy) xw[i00 - dX - dY] = rpd;
            dg[0] = dmx;
            dg[1] = dmy;
            dg[2] = 0.0;
            dg[3] = 1.0;
        }
    }

    // ---------------------------------------------------------------- 2b. own nodes (ROWS rows per warp)
    {
        double *px = xw + WY(t_first) * W + wc;
        double *pw = cW + (WY(t_first) - 2) * T + (wc - 2);
        constexpr int dYw = SY ? -T : T;
        double2 cur = make_double2(0.0, 0.0);
        if constexpr (SOR) cur = *reinterpret_cast<const double2 *>(px);
        auto row = [&](int k, bool last) {
            // faces, global orientation: node 0 = column wc, node 1 = wc + 1
            const double2 fx = rfx[k];
            const double fxn = __shfl_down_sync(0xffffffffu, fx.x, 1);   // all lanes take part
            const double fx2 = (lane == 31) ? rfe[k] : fxn;
            const double2 fn = rfy[k];
            const double2 ylo = SY ? fn : fcarry, yhi = SY ? fcarry : fn;
            fcarry = fn;
            const double xl0 = fx.x, xh0 = fx.y, xl1 = fx.y, xh1 = FACES ? fx2 : 1.0;
            const double2 bb = rb[k];
            double a0, a1, r00, r01;
            if constexpr (SOR) {
                const double2 nb = (last && warp < NW - 1) ? save : *reinterpret_cast<const double2 *>(px + dY);
                double e0, e1;                               // explicit (local +x) neighbours
                if constexpr (SX) {
                    const double up = __shfl_up_sync(0xffffffffu, cur.y, 1);
                    e0 = (lane == 0) ? px[-1] : up;
                    e1 = cur.x;
                } else {
                    const double dn = __shfl_down_sync(0xffffffffu, cur.x, 1);
                    e0 = cur.y;
                    e1 = (lane == 31) ? px[2] : dn;
                }
                const double ap0 = ((xl0 + xh0) + (ylo.x + yhi.x)) + beta;
                const double ap1 = ((xl1 + xh1) + (ylo.y + yhi.y)) + beta;
                a0 = div_rn(w_o, ap0);
                a1 = div_rn(w_o, ap1);
                r00 = fma(a0, fma(SY ? ylo.x : yhi.x, nb.x, fma(SX ? xl0 : xh0, e0, bb.x)), omw * cur.x);
                r01 = fma(a1, fma(SY ? ylo.y : yhi.y, nb.y, fma(SX ? xl1 : xh1, e1, bb.y)), omw * cur.y);
                cur = nb;
            } else {
                const double2 sv = *reinterpret_cast<const double2 *>(px);
                if (invd) {
                    a0 = bb.x;
                    a1 = bb.y;
                } else {
                    a0 = div_rn(w_o, ((xl0 + xh0) + (ylo.x + yhi.x)) + beta);
                    a1 = div_rn(w_o, ((xl1 + xh1) + (ylo.y + yhi.y)) + beta);
                }
                r00 = A.rscale ? a0 * sv.x : A.coef * sv.x;
                r01 = A.rscale ? a1 * sv.y : A.coef * sv.y;
            }
            *reinterpret_cast<double2 *>(px) = make_double2(r00, r01);
            st_shared_v2_noalias(pw, a0 * (SX ? xh0 : xl0), a1 * (SX ? xh1 : xl1));
            st_shared_v2_noalias(pw + NCOEF, a0 * (SY ? yhi.x : ylo.x), a1 * (SY ? yhi.y : ylo.y));
            px += dY;
            pw += dYw;
        };
#pragma unroll 1
        for (int t0 = 0; t0 < ROWS - RING; t0 += RING) {
#pragma unroll
            for (int k = 0; k < RING; ++k) {
                row(k, false);
                if (load_aux) rb[k] = __ldg(reinterpret_cast<const double2 *>(pb));
                if constexpr (FACES) {
                    rfx[k] = __ldg(reinterpret_cast<const double2 *>(pfx));
                    rfe[k] = (lane == 31) ? __ldg(pfx + 2) : 0.0;
                    rfy[k] = __ldg(reinterpret_cast<const double2 *>(pfy));
                }
                pb += rstep;
                pfx += rstep;
                pfy += rstep;
            }
        }
#pragma unroll
        for (int k = 0; k < RING; ++k) row(k, k == RING - 1);
    }
    __syncthreads();
    SW_TMARK(t_prologue);
    if (SW_V2_AHEAD > 0 && threadIdx.x == 64 && AH.tx >= 0) {
        tma_prefetch_2d(AH.x, AH.tx * T, AH.ty * T);
        if (load_aux) tma_prefetch_2d(AH.b, AH.tx * T + 2, AH.ty * T + 2);
        if constexpr (FACES) {
            tma_prefetch_2d(AH.fx, AH.tx * T + 2, AH.ty * T + 2);
            tma_prefetch_2d(AH.fy, AH.tx * T + 2, AH.ty * T + 2);
        }
    }

    // ---------------------------------------------------------------- 3. corner and chains (warp 1)
    if (warp == 1 && lane == 0) {
        if (cx && cy) {
            constexpr int xlo_p = (SX == 0), ylo_p = (SY == 0);
            double M[4][4], rhs[4], uu[4];
            int idx[4];
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                const int isx = (m & 1) ? !xlo_p : xlo_p;
                const int isy = (m & 2) ? !ylo_p : ylo_p;
                idx[m] = i00 - (isx ? dX : 0) - (isy ? dY : 0);
                // coupling of member m to its partner across x (m^1) and across y (m^2)
                const double mxv = (isx && isy) ? dg[0] : (isx ? xch_p[0] : (isy ? ych_c[0] : cW[c00]));
                const double myv = (isx && isy) ? dg[1] : (isx ? xch_c[0] : (isy ? ych_p[0] : cS[c00]));
#pragma unroll
                for (int q = 0; q < 4; ++q) M[m][q] = (m == q) ? 1.0 : 0.0;
                rhs[m] = xw[idx[m]];
                M[m][m ^ 1] = -mxv;
                M[m][m ^ 2] = -myv;
            }
            ge_solve_k<4>(M, rhs, uu, A.flag);
#pragma unroll
            for (int m = 0; m < 4; ++m) xw[idx[m]] = uu[m];
        } else if (cx || cy) {
            const int ip = cx ? i00 - dX : i00 - dY;
            const double m_op = cx ? cW[c00] : cS[c00];          // own -> partner
            const double m_po = cx ? xch_p[0] : ych_p[0];        // partner -> own
            const bool pfirst = cx ? (SX == 0) : (SY == 0);
            double M[2][2], rhs[2], uu[2];
            M[0][0] = M[1][1] = 1.0;
            rhs[0] = pfirst ? xw[ip] : xw[i00];
            rhs[1] = pfirst ? xw[i00] : xw[ip];
            M[0][1] = -(pfirst ? m_po : m_op);
            M[1][0] = -(pfirst ? m_op : m_po);
            ge_solve_k<2>(M, rhs, uu, A.flag);
            xw[i00] = pfirst ? uu[1] : uu[0];
            xw[ip] = pfirst ? uu[0] : uu[1];
        }
    }
    if (warp == 1) {
        // pivots of the chain pairs, all k in parallel: fma(m_ba, -m_ab, 1) is symmetric in the
        // two couplings (exact product), so member order does not matter here
        int fl = 0;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int k = h * 32 + lane;
            const double my = fma(cS[CI(k, 0)], -ych_p[k], 1.0), mx = fma(cW[CI(0, k)], -xch_p[k], 1.0);
            fl |= (cy && !(fabs(my) >= 1e-14)) || (cx && !(fabs(mx) >= 1e-14));
            inv_y[k] = div_rn(1.0, my);
            inv_x[k] = div_rn(1.0, mx);
        }
        if (fl) atomicOr(A.flag, 1);
    }
    __syncwarp();
    SW_TMARK(t_c0);
    if (warp == 1 && lane < 2) {
        // lane 0: chain along local row 0 (pairs with the y-face partners (k,-1));
        // lane 1: chain along local column 0 (pairs with the x-face partners (-1,k)).
        // Member order a = lower global index (oracle ge_solve); an uncoupled face runs the
        // same code with a = the zero ghost node and zero couplings.
        const int step = lane ? dY : dX, cstep = lane ? dYc : dX, perp = lane ? dX : dY;
        const bool coupled = lane ? cx : cy;
        const bool pfirst = lane ? (SX == 0) : (SY == 0);
        const bool a_is_p = pfirst || !coupled;
        const double *oc = (lane ? cS : cW) + c00, *op = (lane ? cW : cS) + c00;   // own: chain / pair coupling
        const double *pc = lane ? xch_c : ych_c, *pp = lane ? xch_p : ych_p;      // partner: chain / pair
        const double *zero = dg + 2;
        // (pointer, stride) of: chain coupling of a and b, pair coupling of a (m_ab) and b (m_ba)
        const double *qa = a_is_p ? (coupled ? pc : zero) : oc;
        const int sa = a_is_p ? (coupled ? 1 : 0) : cstep;
        const double *qb = a_is_p ? oc : pc;
        const int sb = a_is_p ? cstep : 1;
        const double *qab = a_is_p ? (coupled ? pp : zero) : op;
        const double *qba = a_is_p ? (coupled ? op : zero) : pp;
        const int sba = a_is_p ? (coupled ? cstep : 0) : 1;
        const double *qi = coupled ? (lane ? inv_x : inv_y) : dg + 3;
        const int si = coupled ? 1 : 0;
        int ia = a_is_p ? i00 - perp : i00;
        int ib = a_is_p ? i00 : i00 - perp;
        double pa = xw[ia], pb2 = xw[ib];
        // step k+1 operands are loaded before the stores of step k
        double n_ra = xw[ia + step], n_rb = xw[ib + step];
        double n_ma = qa[sa], n_mb = qb[sb], n_mab = qab[sa], n_mba = qba[sba], n_inv = qi[si];
#pragma unroll 2
        for (int k = 1; k < T; ++k) {
            ia += step;
            ib += step;
            const double r0a = n_ra, r0b = n_rb, ma = n_ma, mb = n_mb, mab = n_mab, mba = n_mba, inv1 = n_inv;
            n_ra = xw[ia + step];
            n_rb = xw[ib + step];
            n_ma = qa[(k + 1) * sa];
            n_mb = qb[(k + 1) * sb];
            n_mab = qab[(k + 1) * sa];
            n_mba = qba[(k + 1) * sba];
            n_inv = qi[(k + 1) * si];
            const double ra = fma(ma, pa, r0a);
            const double rb = fma(mb, pb2, r0b);
            pb2 = fma(mba, ra, rb) * inv1;
            pa = fma(mab, pb2, ra);
            xw[ia] = pa;
            xw[ib] = pb2;
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
        const int rA = 2 * lane + 1;
        double *p = xw + WI(1, rA) + (-lane) * dX;         // step 0: c = 1 - lane
        double *q = cW + CI(1, rA) + (-lane) * dX;
        double WA = xw[WI(0, rA)], WB = xw[WI(0, rA) + dY];
        double uBp = 0.0;
        double nr0A = p[0], nr0B = p[dY], nrow0 = p[-rA * dY];
        double nwA = q[0], nwB = q[dYc], nsA = q[NCOEF], nsB = q[NCOEF + dYc];
        auto stepf = [&](int s, int RAMP) {
            const int c = s - lane + 1;
            const bool act = RAMP == 0 ? true : (RAMP == 1 ? c >= 1 : c <= T - 1);
            const double r0A = nr0A, r0B = nr0B, row0 = nrow0, mwA = nwA, mwB = nwB, msA = nsA, msB = nsB;
            double *pn = p + dX;
            const double *qn = q + dX;
            nr0A = pn[0];
            nr0B = pn[dY];
            nrow0 = pn[-rA * dY];
            nwA = qn[0];
            nwB = qn[dYc];
            nsA = qn[NCOEF];
            nsB = qn[NCOEF + dYc];
            const double S = sel_f64(lane == 0, row0, shfl_up1_f64(uBp));
            const double uA = fma(msA, S, fma(mwA, WA, r0A));
            const double nB = fma(msB, uA, fma(mwB, WB, r0B));
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
            p = pn;
            q = const_cast<double *>(qn);
        };
#pragma unroll 4
        for (int s = 0; s < 31; ++s) stepf(s, 1);
#pragma unroll 4
        for (int s = 31; s < 63; ++s) stepf(s, 0);
#pragma unroll 4
        for (int s = 63; s < 94; ++s) stepf(s, 2);
        SW_TMARK(t_w1);
        SW_TADDT(7, t_w0, t_w1, 0);
    }

    // ---------------------------------------------------------------- 5. write-back (ROWS rows per warp)
    __syncthreads();
    SW_TMARK(t_wave);
    {
        const int r0 = 2 + warp * ROWS;
        const double *src = xw + r0 * W + wc;
        double2 *dst = reinterpret_cast<double2 *>(A.xnew + (y0 + r0) * P0 + x0 + wc);
#pragma unroll 8
        for (int r = 0; r < ROWS; ++r) __stcs(dst + r * (P0 / 2), *reinterpret_cast<const double2 *>(src + r * W));
    }
    SW_TMARK(t_end);
    SW_TADD(0, t_start, t_staged);
    SW_TADD(1, t_staged, t_prologue);
    SW_TADD(2, t_prologue, t_chains);
    SW_TADD(3, t_chains, t_wave);
    SW_TADD(4, t_wave, t_end);
    SW_TADD(5, 0, 1);
}

template <int MODE, bool FACES>
__global__ void __launch_bounds__(v2::NW * 32, 2)
    k_sweep2v(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmb,
              const __grid_constant__ CUtensorMap tmfx, const __grid_constant__ CUtensorMap tmfy, Sweep2vArgs A) {
    extern __shared__ __align__(128) double sm[];
    SW_JITTER_POINT();
    __shared__ uint64_t bar;
    const Geo &G = A.G;
    const int tx = blockIdx.x % G.nt[0];
    const int ty = blockIdx.x / G.nt[0];
    const int64_t R0 = tx, R1 = ty + G.toff[1];
    const int sx = ((A.base >> 0) & 1) ^ (int)(R0 & 1);
    const int sy = ((A.base >> 1) & 1) ^ (int)(R1 & 1);
    const bool cx = A.couple && (sx ? (R0 < G.ntg[0] - 1) : (R0 > 0));
    const bool cy = A.couple && (sy ? (R1 < G.ntg[1] - 1) : (R1 > 0));
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
        mbar_expect_tx(&bar, (uint32_t)(sizeof(double) * v2::WS));
        tma_load_2d(sm, &tmx, tx * v2::T, ty * v2::T, &bar);
        if (MODE == MODE_SOR || A.invd_mode) tma_prefetch_2d(&tmb, tx * v2::T + 2, ty * v2::T + 2);
        if (FACES) {
            tma_prefetch_2d(&tmfx, tx * v2::T + 2, ty * v2::T + 2);
            tma_prefetch_2d(&tmfy, tx * v2::T + 2, ty * v2::T + 2);
        }
    }
    __syncthreads();
    Ahead2v AH{&tmx, &tmb, &tmfx, &tmfy, -1, 0};
    if (SW_V2_AHEAD > 0) {
        const int64_t nb = (int64_t)blockIdx.x + SW_V2_AHEAD;
        if (nb < (int64_t)gridDim.x) {
            AH.tx = (int)(nb % G.nt[0]);
            AH.ty = (int)(nb / G.nt[0]);
        }
    }
    switch (sx | (sy << 1)) {
        case 0: sweep2v_tile<MODE, FACES, 0, 0>(A, sm, &bar, tx, ty, cx, cy, AH); break;
        case 1: sweep2v_tile<MODE, FACES, 1, 0>(A, sm, &bar, tx, ty, cx, cy, AH); break;
        case 2: sweep2v_tile<MODE, FACES, 0, 1>(A, sm, &bar, tx, ty, cx, cy, AH); break;
        default: sweep2v_tile<MODE, FACES, 1, 1>(A, sm, &bar, tx, ty, cx, cy, AH); break;
    }
}

template <int MODE, bool FACES>
inline cudaError_t launch_k2v(const CUtensorMap &tmx, const CUtensorMap &tmb, const CUtensorMap &tmfx,
                              const CUtensorMap &tmfy, const Sweep2vArgs &A, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_sweep2v<MODE, FACES>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)v2::SMEM);
        cudaFuncSetAttribute(k_sweep2v<MODE, FACES>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        attr = true;
    }
    const unsigned tiles = (unsigned)((int64_t)A.G.nt[0] * A.G.nt[1]);
    k_sweep2v<MODE, FACES><<<tiles, v2::NW * 32, v2::SMEM, s>>>(tmx, tmb, tmfx, tmfy, A);
    return cudaGetLastError();
}

inline cudaError_t launch_sweep2v(const CUtensorMap &tmx, const CUtensorMap &tmb, const CUtensorMap &tmfx,
                                  const CUtensorMap &tmfy, const Geo &G, int base, const double *w8, const double *b,
                                  const double *fx, const double *fy, double *xn, int *flag, cudaStream_t s) {
    Sweep2vArgs A{};
    A.G = G;
    A.base = base;
    for (int i = 0; i < 4; ++i) A.omega[i] = w8[i];
    A.b = b;
    A.fx = fx;
    A.fy = fy;
    A.xnew = xn;
    A.flag = flag;
    A.couple = 1;
    return launch_k2v<MODE_SOR, true>(tmx, tmb, tmfx, tmfy, A, s);
}

// One block-triangular solve out = (D/alpha + A_I)^-1 r0 over the 64 x 64 boxes at corner bits
// `base` (see MODE_TRI above).  tsrc: 68 x 68 window map of src; taux: 64 x 64 map of 1/D~
// (ILU) for the L2 prefetch; faces may be null (unit coefficients).
inline cudaError_t launch_tri2v(const CUtensorMap &tsrc, const CUtensorMap &taux, const CUtensorMap &tmfx,
                                const CUtensorMap &tmfy, const Geo &G, int base, double omega, const double *invd,
                                const double *fx, const double *fy, bool rscale, double coef, bool couple, double *out,
                                int *flag, cudaStream_t s) {
    Sweep2vArgs A{};
    A.G = G;
    A.base = base;
    for (int i = 0; i < 4; ++i) A.omega[i] = omega;
    A.b = invd;
    A.fx = fx;
    A.fy = fy;
    A.xnew = out;
    A.flag = flag;
    A.coef = coef;
    A.invd_mode = invd != nullptr;
    A.rscale = rscale;
    A.couple = couple;
    if (fx) return launch_k2v<MODE_TRI, true>(tsrc, taux, tmfx, tmfy, A, s);
    return launch_k2v<MODE_TRI, false>(tsrc, taux, tmfx, tmfy, A, s);
}

}  // namespace sw
