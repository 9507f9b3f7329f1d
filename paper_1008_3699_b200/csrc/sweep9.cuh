// sweep9.cuh -- decomposed SOR sweep of the nine-point molecule, 2D (PAPER:702-707:
// "the extension of our algorithm for nine-point or higher order central stencils is straightforward
// ... the size of local systems to be solved will be also increased").  Reading R-N3: a neighbour q
// is implicit (new value) for p iff it lies on the start side of p's box along every axis in which
// they differ -- the paper's rule, extended to the diagonals.  A box then takes W, S, SW new and E,
// N, NE, SE, NW old (SE and NW sit on p's own front), pairs of nodes across coupled start faces are
// solved together as in the five-point sweep, and the four nodes at a start corner form one dense
// 4 x 4 system (the five-point sweep's 4-cycle plus the two diagonals).  Per node the oracle's
// operations in its order (or_sweep9): a_P = ((W + E) + (S + N)) + ((SW + NE) + (SE + NW)) + beta,
// r0 = fma(w / a_P, b + sum_explicit c u_old, (1 - w) u_old), implicit terms and the coupled-set
// elimination (no pivoting, ascending global index) in neighbour order W, E, S, N, SW, SE, NW, NE:
// bitwise equal results.
//
// One CTA of 256 threads per box (T0, T1 <= 64): the old values of the box and its 2-node halo in
// shared memory in LOCAL coordinates (local +a points away from the box's start corner); all threads
// then compute alpha and the explicit part r0 of every node of local [-1, T)^2 (own nodes and partner
// layers) into a second window and an alpha window; front d = x + y of the own nodes: thread t < 64
// takes node (t, d - t) unless it is on a coupled start face (its implicit neighbours are local W,
// S, SW); a third warp solves the front's coupled sets (the x- and y-face pairs, the corner); a named
// barrier of those 96 threads per front; write-back by all threads.  Implicit couplings are read from global memory (L1 / L2).
#pragma once
#include "common.cuh"
#include "sweep2p.cuh"

namespace sw {

namespace s9 {
constexpr int NT = 256;   // threads per CTA: the prologue and write-back by all, the fronts by the first LT
constexpr int LT = 64;    // one thread per box column (T0 <= 64): the nodes outside the coupled sets
constexpr int FT = 96;    // threads on the fronts: LT + one warp for the coupled sets (lanes 0 / 1: the
                          // x- / y-face pair of the front, lane 2: the corner set)
__constant__ int NBX[8] = {-1, 1, 0, 0, -1, 1, -1, 1};
__constant__ int NBY[8] = {0, 0, -1, 1, -1, -1, 1, 1};
}  // namespace s9

struct Sweep9Args {
    Geo G;
    int base;
    double omega[4];
    const double *xo, *b, *f0, *f1;   // padded; f0 / f1 null = unit axis faces
    const double *dd, *da;            // padded diagonal coefficients (corner-indexed, R-N3)
    double *xn;
    int *flag;
};

// region 0: the x_old window over local [-2, T + 2), later the coupled-set coefficients (8 per node
// of the start-face layers, 16 (T0 + T1) doubles) and the fronts' coefficient ring; then (r0, later the new values) over local
// [-2, T + 2) and alpha over local [-1, T)
__host__ __device__ inline int sweep9_r0(int T0, int T1) {
    const int w = (T0 + 4) * (T1 + 4), c = 16 * (T0 + T1) + 8 * 64 * 3;   // + the coefficient ring
    return w > c ? w : c;
}
inline size_t sweep9_smem(const Geo &G) {
    return sizeof(double) * ((size_t)sweep9_r0(G.T[0], G.T[1]) + (size_t)(G.T[0] + 4) * (G.T[1] + 4) +
                             (size_t)(G.T[0] + 1) * (G.T[1] + 1));
}

inline bool sweep9_supported(const Geo &G) {
    return G.dim == 2 && G.T[0] <= s9::LT && G.T[1] <= s9::LT && sweep9_smem(G) <= 227 * 1024;
}

__global__ void __launch_bounds__(s9::NT, 2) k_sweep9(Sweep9Args A) {
    extern __shared__ __align__(16) double s9m[];
    SW_JITTER_POINT();
    const Geo &G = A.G;
    const int T0 = G.T[0], T1 = G.T[1], WX = T0 + 4, AX = T0 + 1;
    double *const XO = s9m, *const XN = s9m + sweep9_r0(T0, T1), *const AW = XN + WX * (T1 + 4);
    const int tx = blockIdx.x % G.nt[0], ty = blockIdx.x / G.nt[0];
    const int64_t R0 = tx, R1 = ty + G.toff[1];
    const int sx = ((A.base >> 0) & 1) ^ (int)(R0 & 1);
    const int sy = ((A.base >> 1) & 1) ^ (int)(R1 & 1);
    const bool cx = sx ? (R0 < G.ntg[0] - 1) : (R0 > 0);
    const bool cy = sy ? (R1 < G.ntg[1] - 1) : (R1 > 0);
    const int64_t X0 = R0 * T0, Y0 = R1 * T1;
    auto gxo = [&](int lx) { return X0 + (sx ? T0 - 1 - lx : lx); };
    auto gyo = [&](int ly) { return Y0 + (sy ? T1 - 1 - ly : ly); };
    auto wi = [&](int lx, int ly) { return (ly + 2) * WX + (lx + 2); };
    auto ai = [&](int lx, int ly) { return (ly + 1) * AX + (lx + 1); };
    auto inside = [&](int64_t gx, int64_t gy) { return gx >= 0 && gx < G.ng[0] && gy >= 0 && gy < G.ng[1]; };
    // coefficient of global neighbour k of global node (gx, gy)
    auto coef = [&](int k, int64_t gx, int64_t gy) -> double {
        const int dx = s9::NBX[k], dy = s9::NBY[k];
        const int64_t cxg = gx + (dx > 0), cyg = gy + (dy > 0);
        if (dy == 0) return A.f0 ? __ldg(A.f0 + gidx(G, cxg, gy, 0)) : 1.0;
        if (dx == 0) return A.f1 ? __ldg(A.f1 + gidx(G, gx, cyg, 0)) : 1.0;
        return __ldg((dx == dy ? A.dd : A.da) + gidx(G, cxg, cyg, 0));
    };
    // start side of the box containing local coordinate l (A starts at local 0 and moves +;
    // every neighbouring box's start side is +); q implicit for p iff on p's start side along every
    // axis where they differ (R-N3)
    auto side = [&](int l, int T) { return (l >= 0 && l < T) ? -1 : +1; };
    auto implicit = [&](int px, int py, int qx, int qy) {
        const int sxp = side(px, T0), syp = side(py, T1);
        const bool okx = qx == px || (sxp < 0 ? qx < px : qx > px);
        const bool oky = qy == py || (syp < 0 ? qy < py : qy > py);
        return okx && oky;
    };
    auto lnb = [&](int p, int kk, int &qx, int &qy, int px, int py) {
        qx = px + (sx ? -s9::NBX[kk] : s9::NBX[kk]);
        qy = py + (sy ? -s9::NBY[kk] : s9::NBY[kk]);
        (void)p;
    };
    SW_TMARK(t_start);
    // ---- stage in the old window (0 outside the domain: Dirichlet data are folded into b)
#pragma unroll 4
    for (int e = threadIdx.x; e < WX * (T1 + 4); e += s9::NT) {
        const int lx = e % WX - 2, ly = e / WX - 2;
        const int64_t gx = gxo(lx), gy = gyo(ly);
        XO[e] = inside(gx, gy) ? __ldg(A.xo + gidx(G, gx, gy, 0)) : 0.0;
    }
    __syncthreads();
    SW_TMARK(t_staged);
    SW_TADD(0, t_start, t_staged);
    // ---- explicit parts of every node of local [-1, T)^2 inside the domain (own nodes and the
    // partner layers): alpha = w / a_P, r0 = fma(alpha, b + sum_explicit c u_old, (1 - w) u_old)
    for (int e = threadIdx.x; e < AX * (T1 + 1); e += s9::NT) {
        const int px = e % AX - 1, py = e / AX - 1;
        const int64_t gx = gxo(px), gy = gyo(py);
        if (!inside(gx, gy)) continue;
        double c8[8];
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) c8[kk] = coef(kk, gx, gy);
        const double bv = __ldg(A.b + gidx(G, gx, gy, 0));
        const double ap = ((c8[0] + c8[1]) + (c8[2] + c8[3])) + ((c8[4] + c8[7]) + (c8[5] + c8[6])) + G.beta;
        const int bits = (sx ^ (px < 0 ? 1 : 0)) | ((sy ^ (py < 0 ? 1 : 0)) << 1);
        const double w = A.omega[bits];
        const double al = div_rn(w, ap);
        double ev = bv;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
            if (!inside(gx + s9::NBX[kk], gy + s9::NBY[kk])) continue;
            int qx, qy;
            lnb(0, kk, qx, qy, px, py);
            if (implicit(px, py, qx, qy)) continue;
            ev = fma(c8[kk], XO[wi(qx, qy)], ev);
        }
        XN[wi(px, py)] = fma(al, ev, (1.0 - w) * XO[wi(px, py)]);
        AW[ai(px, py)] = al;
    }
    __syncthreads();
    SW_TMARK(t_r0);
    SW_TADD(1, t_staged, t_r0);
    // ---- the 8 coefficients of every node that can be in a coupled set (local x in {-1, 0} or
    // local y in {-1, 0}), into the x_old window's space (dead from here on)
    const int nslot = 2 * (T1 + 1) + 2 * (T0 - 1);
    double *const CS = XO;
    auto slot = [&](int lx, int ly) {
        return lx <= 0 ? (lx + 1) * (T1 + 1) + (ly + 1) : 2 * (T1 + 1) + (ly + 1) * (T0 - 1) + (lx - 1);
    };
    for (int e = threadIdx.x; e < nslot * 8; e += s9::NT) {
        const int sl = e >> 3, kk = e & 7;
        int lx, ly;
        if (sl < 2 * (T1 + 1)) {
            lx = sl / (T1 + 1) - 1;
            ly = sl % (T1 + 1) - 1;
        } else {
            const int r = sl - 2 * (T1 + 1);
            lx = r % (T0 - 1) + 1;
            ly = r / (T0 - 1) - 1;
        }
        const int64_t gx = gxo(lx), gy = gyo(ly);
        CS[e] = inside(gx, gy) ? coef(kk, gx, gy) : 0.0;
    }
    __syncthreads();
    SW_TMARK(t_cs);
    SW_TADD(2, t_r0, t_cs);
    if (threadIdx.x >= s9::FT) {            // the other warps rejoin for the write-back
        __syncthreads();
        for (int e = threadIdx.x; e < T0 * T1; e += s9::NT) {
            const int lx = e % T0, ly = e / T0;
            A.xn[gidx(G, gxo(lx), gyo(ly), 0)] = XN[wi(lx, ly)];
        }
        return;
    }
    const int t = threadIdx.x;
    int fl = 0;
    // implicit neighbours of an own node outside the sets: local W, S, SW, always in this order in
    // the oracle's global neighbour order.  Their coefficients arrive PD fronts ahead by cp.async
    // into a per-thread ring in region 0 (after the set coefficients): one commit group per front
    const int kW = sx ? 1 : 0, kS = sy ? 3 : 2, kSW = 4 + sx + 2 * sy;
    constexpr int PD = 8;
    double *const RING = XO + 16 * (T0 + T1);                 // [PD][LT][3]
    auto cptr = [&](int k, int64_t gx, int64_t gy) -> const double * {   // address of coef(k, gx, gy)
        const int dx = s9::NBX[k], dy = s9::NBY[k];
        const int64_t cxg = gx + (dx > 0), cyg = gy + (dy > 0);
        if (dy == 0) return A.f0 ? A.f0 + gidx(G, cxg, gy, 0) : nullptr;
        if (dx == 0) return A.f1 ? A.f1 + gidx(G, gx, cyg, 0) : nullptr;
        return (dx == dy ? A.dd : A.da) + gidx(G, cxg, cyg, 0);
    };
    auto fetch = [&](int yy) {                                 // node (t, yy) into slot yy % PD, then commit
        if (t < T0 && yy < T1) {
            const int64_t gx = gxo(t), gy = gyo(yy);
            double *dst = RING + ((yy % PD) * s9::LT + t) * 3;
            const int kk[3] = {kW, kS, kSW};
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                const double *src = cptr(kk[q], gx, gy);
                if (src)
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst + q)), "l"(src) : "memory");
                else
                    dst[q] = 1.0;
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    if (t < s9::LT)
        for (int yy = 0; yy < PD; ++yy) fetch(yy);
    for (int d = 0; d <= (T0 - 1) + (T1 - 1); ++d) {
        // fronts: threads < LT the nodes outside the coupled sets (one branch-free path); one more
        // warp the sets of the front, so the two kinds never diverge inside a warp
        const int x = t < s9::LT ? t : ((t - s9::LT) == 1 ? d : 0);
        const int y = t < s9::LT ? d - t : ((t - s9::LT) == 1 ? 0 : d);
        const bool member = (x == 0 && cx) || (y == 0 && cy);
        const int lane = t - s9::LT;
        const bool valid = x < T0 && y >= 0 && y < T1 &&
                           (t < s9::LT ? !member
                                       : (lane == 0 ? (cx && !(d == 0 && cy))
                                                    : (lane == 1 ? (cy && !(d == 0 && cx)) : (lane == 2 && d == 0 && cx && cy))));
        if (valid) {
            const bool corner = x == 0 && y == 0 && cx && cy;
            const bool xpair = !corner && x == 0 && cx, ypair = !corner && !xpair && y == 0 && cy;
            const int k = corner ? 4 : ((xpair || ypair) ? 2 : 1);
            if (k == 1) {
                // (a neighbour outside the domain holds 0 and is skipped, as in the oracle)
                asm volatile("cp.async.wait_group %0;" ::"n"(PD - 1) : "memory");   // node (t, y)'s group
                const double *cr = RING + ((y % PD) * s9::LT + t) * 3;
                const double cw0 = cr[0], cs0 = cr[1], cd0 = cr[2];
                const int64_t gx = gxo(x), gy = gyo(y);
                const double al = AW[ai(x, y)];
                double acc = XN[wi(x, y)];
                if (inside(gx + s9::NBX[kW], gy)) acc = fma(al * cw0, XN[wi(x - 1, y)], acc);
                if (inside(gx, gy + s9::NBY[kS])) acc = fma(al * cs0, XN[wi(x, y - 1)], acc);
                if (inside(gx + s9::NBX[kSW], gy + s9::NBY[kSW])) acc = fma(al * cd0, XN[wi(x - 1, y - 1)], acc);
                XN[wi(x, y)] = acc;
            } else if (k == 2) {
                // a pair across one coupled start face, in registers: members in ascending global
                // index, rows (1, -m01; -m10, 1), the oracle's ge_solve for K = 2 written out
                const int px2 = xpair ? -1 : x, py2 = xpair ? y : -1;
                const bool sw01 = gyo(py2) * G.ng[0] + gxo(px2) < gyo(y) * G.ng[0] + gxo(x);
                const int ax = sw01 ? px2 : x, ay = sw01 ? py2 : y;
                const int bx = sw01 ? x : px2, by = sw01 ? y : py2;
                auto row = [&](int px, int py, int ox, int oy, double &moff) {
                    const int64_t gx = gxo(px), gy = gyo(py);
                    const double al = AW[ai(px, py)];
                    const double *cs = CS + 8 * slot(px, py);
                    double acc = XN[wi(px, py)];
                    moff = 0.0;
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) {
                        if (!inside(gx + s9::NBX[kk], gy + s9::NBY[kk])) continue;
                        int qx, qy;
                        lnb(0, kk, qx, qy, px, py);
                        if (!implicit(px, py, qx, qy)) continue;
                        const double m = al * cs[kk];
                        if (qx == ox && qy == oy) moff = -m;
                        else acc = fma(m, XN[wi(qx, qy)], acc);
                    }
                    return acc;
                };
                double m01, m10, r0a, r0b;
                if (d >= 1) {
                    // a chain pair (d >= 1), its rows written out: besides the member across the face,
                    // the own node's implicit neighbours are the previous chain node (along the face)
                    // and the previous partner (diagonal), the partner's are the previous partner and
                    // the previous chain node (diagonal); in the oracle's global neighbour order the
                    // axis neighbour comes before the diagonal, so acc = fma(diag, ., fma(axis, ., r0))
                    const int ox = x, oy = y;                              // own node
                    const int dxl = xpair ? 0 : -1, dyl = xpair ? -1 : 0;  // local step back along the chain
                    const int kax = xpair ? (sy ? 3 : 2) : (sx ? 1 : 0);   // the axis step back (S / W)
                    const int kd_o = 4 + sx + 2 * sy;                      // own: local SW
                    // partner: local SW seen from the other side (x-face: SE; y-face: NW)
                    const int kd_p = xpair ? 4 + (sx ^ 1) + 2 * sy : 4 + sx + 2 * (sy ^ 1);
                    const int kc_o = xpair ? (sx ? 1 : 0) : (sy ? 3 : 2);  // own -> partner (local W / S)
                    const int kc_p = xpair ? (sx ? 0 : 1) : (sy ? 2 : 3);  // partner -> own (local E / N)
                    const double al_o = AW[ai(ox, oy)], al_p = AW[ai(px2, py2)];
                    const double *cs_o = CS + 8 * slot(ox, oy), *cs_p = CS + 8 * slot(px2, py2);
                    const double u_op = XN[wi(ox + dxl, oy + dyl)], u_pp = XN[wi(px2 + dxl, py2 + dyl)];
                    const double acc_o = fma(al_o * cs_o[kd_o], u_pp, fma(al_o * cs_o[kax], u_op, XN[wi(ox, oy)]));
                    const double acc_p = fma(al_p * cs_p[kd_p], u_op, fma(al_p * cs_p[kax], u_pp, XN[wi(px2, py2)]));
                    const double mo = -(al_o * cs_o[kc_o]), mp = -(al_p * cs_p[kc_p]);
                    r0a = sw01 ? acc_p : acc_o;
                    r0b = sw01 ? acc_o : acc_p;
                    m01 = sw01 ? mp : mo;
                    m10 = sw01 ? mo : mp;
                } else {
                    r0a = row(ax, ay, bx, by, m01);
                    r0b = row(bx, by, ax, ay, m10);
                }
                const double inv0 = div_rn(1.0, 1.0);
                const double l = m10 * inv0;
                const double m11 = fma(-l, m01, 1.0);
                const double rb = fma(-l, r0a, r0b);
                fl |= !(fabs(m11) >= 1e-14);
                const double inv1 = div_rn(1.0, m11);
                const double ub = rb * inv1;
                const double ua = fma(-m01, ub, r0a) * inv0;
                XN[wi(ax, ay)] = ua;
                XN[wi(bx, by)] = ub;
            } else {
                // the corner set: the four start-corner nodes, a dense 4 x 4 (once per box)
                int mx[4] = {0, -1, 0, -1}, my[4] = {0, 0, -1, -1};
                int64_t gi[4];
                for (int m = 0; m < k; ++m) gi[m] = gyo(my[m]) * G.ng[0] + gxo(mx[m]);
                for (int a1 = 1; a1 < k; ++a1)
                    for (int b1 = a1; b1 > 0 && gi[b1 - 1] > gi[b1]; --b1) {
                        int64_t tg = gi[b1]; gi[b1] = gi[b1 - 1]; gi[b1 - 1] = tg;
                        int tt = mx[b1]; mx[b1] = mx[b1 - 1]; mx[b1 - 1] = tt;
                        tt = my[b1]; my[b1] = my[b1 - 1]; my[b1 - 1] = tt;
                    }
                double M[4][4], rhs[4], u[4];
                for (int p = 0; p < k; ++p) {
                    const int px = mx[p], py = my[p];
                    const int64_t gx = gxo(px), gy = gyo(py);
                    const double al = AW[ai(px, py)];
                    double acc = XN[wi(px, py)];
                    for (int q = 0; q < k; ++q) M[p][q] = (p == q) ? 1.0 : 0.0;
                    const double *cs = CS + 8 * slot(px, py);
                    for (int kk = 0; kk < 8; ++kk) {
                        if (!inside(gx + s9::NBX[kk], gy + s9::NBY[kk])) continue;
                        int qx, qy;
                        lnb(0, kk, qx, qy, px, py);
                        if (!implicit(px, py, qx, qy)) continue;
                        const double m = al * cs[kk];
                        int in = -1;
                        for (int q = 0; q < k; ++q)
                            if (mx[q] == qx && my[q] == qy) in = q;
                        if (in >= 0) M[p][in] = -m;
                        else acc = fma(m, XN[wi(qx, qy)], acc);
                    }
                    rhs[p] = acc;
                }
                double inv[4];                             // the oracle's ge_solve (R-8)
                for (int p = 0; p < k; ++p) {
                    const double piv = M[p][p];
                    fl |= !(fabs(piv) >= 1e-14);
                    inv[p] = div_rn(1.0, piv);
                    for (int q = p + 1; q < k; ++q) {
                        const double l = M[q][p] * inv[p];
                        for (int j = p + 1; j < k; ++j) M[q][j] = fma(-l, M[p][j], M[q][j]);
                        rhs[q] = fma(-l, rhs[p], rhs[q]);
                    }
                }
                for (int p = k - 1; p >= 0; --p) {
                    double sacc = rhs[p];
                    for (int j = p + 1; j < k; ++j) sacc = fma(-M[p][j], u[j], sacc);
                    u[p] = sacc * inv[p];
                }
                for (int m = 0; m < k; ++m) XN[wi(mx[m], my[m])] = u[m];
            }
        }
        if (t < s9::LT && x < T0 && y >= 0 && y < T1) {   // this slot is read: refill it PD rows ahead
            if (!valid) asm volatile("cp.async.wait_group %0;" ::"n"(PD - 1) : "memory");   // (keep the count)
            fetch(y + PD);
        }
        asm volatile("bar.sync 1, %0;" ::"r"(s9::FT) : "memory");
        SW_JITTER_POINT();
    }
    if (fl) atomicOr(A.flag, 1);
    SW_TMARK(t_fronts);
    SW_TADD(3, t_cs, t_fronts);
    SW_TADD(5, 0, 1);
    __syncthreads();                          // with the waiting warps
    for (int e = threadIdx.x; e < T0 * T1; e += s9::NT) {
        const int lx = e % T0, ly = e / T0;
        A.xn[gidx(G, gxo(lx), gyo(ly), 0)] = XN[wi(lx, ly)];
    }
}

inline cudaError_t launch_sweep9(const Sweep9Args &A, cudaStream_t s) {
    const size_t sm = sweep9_smem(A.G);
    static size_t attr = 0;
    if (sm > attr) {
        cudaFuncSetAttribute(k_sweep9, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        attr = sm;
    }
    const unsigned tiles = (unsigned)((int64_t)A.G.nt[0] * A.G.nt[1]);
    k_sweep9<<<tiles, s9::NT, sm, s>>>(A);
    return cudaGetLastError();
}

}  // namespace sw
