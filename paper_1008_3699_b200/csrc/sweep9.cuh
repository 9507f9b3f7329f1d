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
// One CTA of 256 threads per box (T0, T1 <= 64), two CTAs per SM:
//  1. the old values of the box and its 2-node halo into shared memory in LOCAL coordinates (local +a
//     points away from the box's start corner);
//  2. all threads: alpha and the explicit part r0 of every node of local [-1, T)^2 (own nodes and the
//     partner layers), three nodes per thread and pass with all their global loads in flight;
//  3. threads 0..127: per step of the two start-face chains the pair data (implicit couplings of both
//     members, the 2 x 2 matrix in the oracle's member order and its pivot reciprocal); thread 0: the
//     start corner (the dense 4 x 4, or a pair);
//  4. warp 0, lanes 0 / 1: the chains of 2 x 2 systems along local row 0 / column 0 (or the plain
//     recurrence along a physical boundary), then the whole warp: the wavefront over [1, T)^2 as in
//     k_sweep2p -- lane l owns rows 2l+1, 2l+2, S by shfl.up, W and SW from registers; the nodes'
//     three implicit coefficients come from a shared-memory ring that warps 1..7 fill a chunk of
//     8 steps ahead (coalesced row segments, one named barrier per chunk);
//  5. write-back by all threads.
#pragma once
#include <type_traits>

#include "common.cuh"
#include "sweep2p.cuh"

namespace sw {

namespace s9 {
constexpr int NT = 256;   // threads per CTA
constexpr int PD = 16;    // wavefront coefficient ring depth (steps ahead)
constexpr int CDW = 8;    // doubles of chain data per chain step
// ring element (slot, coefficient j, lane): slot * RSL + j * RJL + lane.  The wavefront reads one
// (slot, j) for all lanes (consecutive words); a producer warp stores 8 consecutive slots x 4
// coefficients of one lane: with RJL = 33, RSL = 198 (= 6 mod 16) a half-warp's 16 stores fall into
// 16 different 8-byte banks.
constexpr int RJL = 33, RSL = 6 * RJL;
constexpr int NPROD = NT - 32;   // producer threads (warps 1..7)
__constant__ int NBX[8] = {-1, 1, 0, 0, -1, 1, -1, 1};   // global neighbour order W, E, S, N, SW, SE, NW, NE
__constant__ int NBY[8] = {0, 0, -1, 1, -1, -1, 1, 1};
__host__ __device__ constexpr int nbx(int k) { return k == 0 ? -1 : (k == 1 ? 1 : (k < 4 ? 0 : ((k & 1) ? 1 : -1))); }
__host__ __device__ constexpr int nby(int k) { return k < 2 ? 0 : (k == 2 ? -1 : (k == 3 ? 1 : (k < 6 ? -1 : 1))); }
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

// region 0: the x_old window over local [-2, T + 2), after the explicit parts the chain data
// [2][64][CDW], the wavefront's coefficient ring [PD][32][6] and the corner's 4 x 8 coefficients; then (r0, later the new values) over
// local [-2, T + 2) and alpha over local [-1, T)
__host__ __device__ inline int sweep9_r0(int T0, int T1) {
    const int w = (T0 + 4) * (T1 + 4), c = 2 * 64 * s9::CDW + s9::PD * s9::RSL + 32;
    return w > c ? w : c;
}
inline size_t sweep9_smem(const Geo &G) {
    return sizeof(double) * ((size_t)sweep9_r0(G.T[0], G.T[1]) + (size_t)(G.T[0] + 4) * (G.T[1] + 4) +
                             (size_t)(G.T[0] + 1) * (G.T[1] + 1));
}

inline bool sweep9_supported(const Geo &G) {
    return G.dim == 2 && G.T[0] <= 64 && G.T[1] <= 64 && sweep9_smem(G) <= 227 * 1024;
}

// TC > 0: square boxes of TC nodes an axis, known at compile time (the index arithmetic of the
// stage-in, the explicit parts and the write-back then needs no runtime division); TC = 0: any box.
#ifndef SW_S9_AHEAD
#define SW_S9_AHEAD 222
#endif
#ifndef SW_S9_AHEAD_AT
#define SW_S9_AHEAD_AT 1      // the chunk after which the producers issue the look-ahead prefetches
#endif
template <int TC>
__global__ void __launch_bounds__(s9::NT, 2) k_sweep9(Sweep9Args A) {
    extern __shared__ __align__(16) double s9m[];
    SW_JITTER_POINT();
    const Geo &G = A.G;
    const int T0 = TC ? TC : G.T[0], T1 = TC ? TC : G.T[1], WX = T0 + 4, AX = T0 + 1;
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
    // partner layers): alpha = w / a_P, r0 = fma(alpha, b + sum_explicit c u_old, (1 - w) u_old).
    // Three nodes per thread and pass, all 27 of their global loads issued before any use; the
    // box's directions are compile-time constants of one of four instantiations (the implicit /
    // explicit split and the window offsets of the neighbours fold away).
    auto explicit_parts = [&](auto SXc, auto SYc) {
        constexpr int SX = decltype(SXc)::value, SY = decltype(SYc)::value;
        const int NA = AX * (T1 + 1);
        const int64_t ng0 = G.ng[0], ng1 = G.ng[1], P0 = G.P0;
        const int64_t gx0 = SX ? X0 + T0 - 1 : X0, gy0 = SY ? Y0 + T1 - 1 : Y0;   // global of local (0, 0)
        constexpr int SGX = SX ? -1 : 1, SGY = SY ? -1 : 1;
        const int dq = 3 * s9::NT / AX, dr = 3 * s9::NT % AX;                     // pass stride in (row, column)
        int qx = threadIdx.x % AX, qy = threadIdx.x / AX;                         // first node of this thread
        for (int e0 = threadIdx.x; e0 < NA; e0 += 3 * s9::NT) {
            double c8[3][8], bv[3];
            int px[3], py[3];
            int64_t gx[3], gy[3];
            bool ok[3];
#pragma unroll
            for (int u = 0; u < 3; ++u) {
                const int e = e0 + u * s9::NT;
                const int ex = qx + (u * s9::NT) % AX, ey = qy + (u * s9::NT) / AX;   // (one carry at most)
                px[u] = (ex >= AX ? ex - AX : ex) - 1;
                py[u] = (ex >= AX ? ey + 1 : ey) - 1;
                gx[u] = gx0 + SGX * px[u];
                gy[u] = gy0 + SGY * py[u];
                ok[u] = e < NA && gx[u] >= 0 && gx[u] < ng0 && gy[u] >= 0 && gy[u] < ng1;
                // coefficient of global neighbour k (coef(), R-N3): faces at the node (W, S) or
                // one step up (E, N), diagonals at the cell corners
                const int64_t i = ok[u] ? gidx(G, gx[u], gy[u], 0) : G.origin;
                c8[u][0] = A.f0 ? __ldg(A.f0 + i) : 1.0;
                c8[u][1] = A.f0 ? __ldg(A.f0 + i + 1) : 1.0;
                c8[u][2] = A.f1 ? __ldg(A.f1 + i) : 1.0;
                c8[u][3] = A.f1 ? __ldg(A.f1 + i + P0) : 1.0;
                c8[u][4] = __ldg(A.dd + i);
                c8[u][5] = __ldg(A.da + i + 1);
                c8[u][6] = __ldg(A.da + i + P0);
                c8[u][7] = __ldg(A.dd + i + 1 + P0);
                bv[u] = __ldg(A.b + i);
            }
            qx += dr;
            qy += dq;
            if (qx >= AX) {
                qx -= AX;
                ++qy;
            }
#pragma unroll
            for (int u = 0; u < 3; ++u) {
                if (!ok[u]) continue;
                const double *c = c8[u];
                const double ap = ((c[0] + c[1]) + (c[2] + c[3])) + ((c[4] + c[7]) + (c[5] + c[6])) + G.beta;
                const int bx = px[u] < 0, by = py[u] < 0;   // partner layers: the neighbour box starts toward ours
                const double w = A.omega[(SX ^ bx) | ((SY ^ by) << 1)];
                const double al = div_rn(w, ap);
                const bool xm = gx[u] > 0, xp = gx[u] + 1 < ng0, ym = gy[u] > 0, yp = gy[u] + 1 < ng1;
                const double *xo = XO + wi(px[u], py[u]);
                double ev = bv[u];
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const int dx = s9::nbx(kk), dy = s9::nby(kk);
                    const bool in = (dx < 0 ? xm : (dx > 0 ? xp : true)) && (dy < 0 ? ym : (dy > 0 ? yp : true));
                    const int ldx = SX ? -dx : dx, ldy = SY ? -dy : dy;
                    // implicit iff on the start side of the node's box along every axis where they
                    // differ (own box: local -; a partner layer's box: local +)
                    const bool impx = dx == 0 || (ldx < 0 ? !bx : bx);
                    const bool impy = dy == 0 || (ldy < 0 ? !by : by);
                    if (in && !(impx && impy)) ev = fma(c[kk], xo[ldx + ldy * WX], ev);
                }
                XN[wi(px[u], py[u])] = fma(al, ev, (1.0 - w) * xo[0]);
                AW[ai(px[u], py[u])] = al;
            }
        }
    };
    switch (sx | (sy << 1)) {
    case 0: explicit_parts(std::integral_constant<int, 0>{}, std::integral_constant<int, 0>{}); break;
    case 1: explicit_parts(std::integral_constant<int, 1>{}, std::integral_constant<int, 0>{}); break;
    case 2: explicit_parts(std::integral_constant<int, 0>{}, std::integral_constant<int, 1>{}); break;
    default: explicit_parts(std::integral_constant<int, 1>{}, std::integral_constant<int, 1>{}); break;
    }
    __syncthreads();
    SW_TMARK(t_r0);
    SW_TADD(1, t_staged, t_r0);
    // ---- region 0 is dead from here on: the chain data and the wavefront's coefficient ring
    double *const CD = XO;                                     // [2][64][CDW]
    double *const RING = XO + 2 * 64 * s9::CDW;                // [PD][32][6]
    double *const CC = RING + s9::PD * s9::RSL;                // corner coefficients [4][8]
    const int lane = threadIdx.x & 31;
    // wavefront geometry (warp 0): lane l owns rows A = 2l + 1 and B = 2l + 2 (local y) and at step
    // s updates column x = s - l + 1 of both; rows >= T1 do not exist
    const int rA = 2 * lane + 1, rB = rA + 1;
    const bool onA = rA < T1, onB = rB < T1;
    const int rAl = onA ? rA : T1 - 1, rBl = onB ? rB : (T1 > 1 ? T1 - 1 : 0);
    // the implicit couplings of a wavefront node are local W, S, SW (global kW, kS, kSW: in the
    // oracle's neighbour order always in this order)
    const int64_t P0 = G.P0;
    const double *const fdg = (sx == sy) ? A.dd : A.da;
    // The coefficients of step s (node column x = s - l + 1 of lane l's rows A and B: W, S, SW of A,
    // then of B; 1.0 for unit faces) live in slot s % PD of the ring, PD = two chunks of CH steps.
    // Warps 1..7 fill it a chunk ahead of the wavefront while warp 0 runs the chains and the fronts
    // (one named barrier of the CTA per chunk): consecutive threads take consecutive columns of one
    // row, so a chunk's 64-byte row segments are read whole instead of one node per lane and step.
    constexpr int CH = s9::PD / 2;
    // hand-off of ring half h (chunks c with c % 2 = h): named barriers FULL[h] = 1 + h (the producer
    // warps arrive when a chunk is stored, the wavefront warp waits before it reads the chunk) and
    // EMPTY[h] = 3 + h (the wavefront warp arrives when it has read the chunk, the producers wait
    // before they overwrite the half)
    auto bar_cnt = [](int) { return 32 + s9::NPROD; };
    auto bar_wait = [&](int id, int cnt) {
        asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(cnt) : "memory");
        SW_JITTER_POINT();
    };
    auto bar_arrive = [&](int id, int cnt) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(cnt) : "memory"); };
    int fl = 0;
    // ---- the chain data (threads 0..127, item (chain, k)): chain 0 = local row 0 (node (k, 0),
    // partner (k, -1) across the y start face), chain 1 = local column 0 (node (0, k), partner
    // (-1, k)).  Besides the member across the face, the own node's implicit neighbours are the
    // previous chain node (axis) and the previous partner (diagonal), the partner's the previous
    // partner (axis) and the previous chain node (diagonal); in the oracle's neighbour order the
    // axis term comes first.  Stored: m_ax, m_d of both, the pair matrix (1, -m01; -m10, 1) in
    // ascending global index and its second pivot's reciprocal (the oracle's ge_solve for K = 2:
    // the first pivot is 1).  An uncoupled face (physical boundary) leaves the plain recurrence
    // along the chain (the other implicit neighbours lie outside the domain).
    if (threadIdx.x < 128) {
        const int ch = threadIdx.x >> 6, k = threadIdx.x & 63;
        const bool cpl = ch == 0 ? cy : cx;
        const int len = ch == 0 ? T0 : T1;
        if (k >= 1 && k < len) {
            const int ox = ch == 0 ? k : 0, oy = ch == 0 ? 0 : k;
            const int kax = ch == 0 ? (sx ? 1 : 0) : (sy ? 3 : 2);        // local W / S
            const int64_t gox = gxo(ox), goy = gyo(oy);
            const double al_o = AW[ai(ox, oy)];
            double *cd = CD + (ch * 64 + k) * s9::CDW;
            cd[0] = al_o * coef(kax, gox, goy);
            if (cpl) {
                const int qx = ch == 0 ? k : -1, qy = ch == 0 ? -1 : k;
                const int kd_o = 4 + sx + 2 * sy;                             // own: local SW
                // partner: local SW seen from the other side (row chain: NW; column chain: SE)
                const int kd_p = ch == 1 ? 4 + (sx ^ 1) + 2 * sy : 4 + sx + 2 * (sy ^ 1);
                const int kc_o = ch == 1 ? (sx ? 1 : 0) : (sy ? 3 : 2);      // own -> partner (local W / S)
                const int kc_p = ch == 1 ? (sx ? 0 : 1) : (sy ? 2 : 3);      // partner -> own (local E / N)
                const int64_t gqx = gxo(qx), gqy = gyo(qy);
                const double al_p = AW[ai(qx, qy)];
                cd[1] = al_o * coef(kd_o, gox, goy);
                cd[2] = al_p * coef(kax, gqx, gqy);
                cd[3] = al_p * coef(kd_p, gqx, gqy);
                const double mo = -(al_o * coef(kc_o, gox, goy)), mp = -(al_p * coef(kc_p, gqx, gqy));
                const bool pfirst = ch == 0 ? (sy == 0) : (sx == 0);          // partner before own
                const double m01 = pfirst ? mp : mo, m10 = pfirst ? mo : mp;
                const double m11 = fma(-m10, m01, 1.0);                       // l = m10 / 1
                fl |= !(fabs(m11) >= 1e-14);
                cd[4] = m01;
                cd[5] = m10;
                cd[6] = div_rn(1.0, m11);
            } else {
                cd[1] = cd[2] = cd[3] = cd[4] = cd[5] = 0.0;
                cd[6] = 1.0;
            }
        }
    }
    // ---- the start corner (warp 4, while warps 0..3 prepare the chain data): the dense 4 x 4 set,
    // a pair across the one coupled face, or a single node without implicit neighbours in the
    // domain (u = r0, nothing to do).  The lanes stage the members' coefficients (member
    // m = (-(m & 1), -(m >> 1)), neighbour k), lane 0 solves.
    if (threadIdx.x >= 128 && threadIdx.x < 160 && (cx || cy)) {
        CC[lane] = coef(lane & 7, gxo(-((lane >> 3) & 1)), gyo(-(lane >> 4)));
        __syncwarp();
        SW_JITTER_POINT();
    }
    if (threadIdx.x == 128 && (cx || cy)) {
        if (cx && cy) {
            constexpr int k = 4;
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
                for (int kk = 0; kk < 8; ++kk) {
                    if (!inside(gx + s9::NBX[kk], gy + s9::NBY[kk])) continue;
                    int qx, qy;
                    lnb(0, kk, qx, qy, px, py);
                    if (!implicit(px, py, qx, qy)) continue;
                    const double m = al * CC[8 * (-px - 2 * py) + kk];
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
        } else {
            // a pair across one coupled start face: members in ascending global index, rows
            // (1, -m01; -m10, 1), the oracle's ge_solve for K = 2 written out
            const int px2 = cx ? -1 : 0, py2 = cx ? 0 : -1;
            const bool sw01 = gyo(py2) * G.ng[0] + gxo(px2) < gyo(0) * G.ng[0] + gxo(0);
            const int ax = sw01 ? px2 : 0, ay = sw01 ? py2 : 0;
            const int bx = sw01 ? 0 : px2, by = sw01 ? 0 : py2;
            auto row = [&](int px, int py, int ox, int oy, double &moff) {
                const int64_t gx = gxo(px), gy = gyo(py);
                const double al = AW[ai(px, py)];
                double acc = XN[wi(px, py)];
                moff = 0.0;
                for (int kk = 0; kk < 8; ++kk) {
                    if (!inside(gx + s9::NBX[kk], gy + s9::NBY[kk])) continue;
                    int qx, qy;
                    lnb(0, kk, qx, qy, px, py);
                    if (!implicit(px, py, qx, qy)) continue;
                    const double m = al * CC[8 * (-px - 2 * py) + kk];
                    if (qx == ox && qy == oy) moff = -m;
                    else acc = fma(m, XN[wi(qx, qy)], acc);
                }
                return acc;
            };
            double m01, m10;
            const double r0a = row(ax, ay, bx, by, m01);
            const double r0b = row(bx, by, ax, ay, m10);
            const double m11 = fma(-m10, m01, 1.0);
            fl |= !(fabs(m11) >= 1e-14);
            const double ub = fma(-m10, r0a, r0b) * div_rn(1.0, m11);
            XN[wi(ax, ay)] = fma(-m01, ub, r0a);
            XN[wi(bx, by)] = ub;
        }
    }
    __syncthreads();
    SW_TMARK(t_cs);
    SW_TADD(2, t_r0, t_cs);
    if (threadIdx.x < 32) {
        // ---- the two start-face chains (lane 0: row 0, lane 1: column 0), then the wavefront
        if (lane < 2) {
            const int ch = lane;
            const bool cpl = ch == 0 ? cy : cx;
            const int len = ch == 0 ? T0 : T1;
            const bool pfirst = ch == 0 ? (sy == 0) : (sx == 0);
            const int so = ch == 0 ? 1 : WX, sp = ch == 0 ? -WX : -1;   // window strides along / across
            double *const xc = XN + wi(0, 0);
            double u_op = xc[0], u_pp = cpl ? xc[sp] : 0.0;             // the corner's results
            const double *const cd = CD + ch * 64 * s9::CDW;
            // the operands of step k + 1 are loaded before the store of step k (off the dependent chain)
            const int k1 = len > 1 ? 1 : 0;
            double n_r0o = xc[k1 * so], n_r0p = cpl ? xc[k1 * so + sp] : 0.0, n_c[7];
#pragma unroll
            for (int j = 0; j < 7; ++j) n_c[j] = cd[k1 * s9::CDW + j];
#pragma unroll 2
            for (int k = 1; k < len; ++k) {
                const double r0o = n_r0o, r0p = n_r0p;
                double c[7];
#pragma unroll
                for (int j = 0; j < 7; ++j) c[j] = n_c[j];
                const int kn = k + 1 < len ? k + 1 : k;
                n_r0o = xc[kn * so];
                n_r0p = cpl ? xc[kn * so + sp] : 0.0;
#pragma unroll
                for (int j = 0; j < 7; ++j) n_c[j] = cd[kn * s9::CDW + j];
                const double in_o = fma(c[0], u_op, r0o);
                const double acc_o = fma(c[1], u_pp, in_o);
                const double acc_p = fma(c[3], u_op, fma(c[2], u_pp, r0p));
                const double r0a = pfirst ? acc_p : acc_o, r0b = pfirst ? acc_o : acc_p;
                const double ub = fma(-c[5], r0a, r0b) * c[6];
                const double ua = fma(-c[4], ub, r0a);
                const double uo = cpl ? (pfirst ? ub : ua) : in_o;
                u_pp = pfirst ? ua : ub;
                u_op = uo;
                xc[k * so] = uo;
            }
        }
        __syncwarp();
        SW_JITTER_POINT();
        SW_TMARK(t_ch);
        SW_TADD(4, t_cs, t_ch);
        // ---- the wavefront over local [1, T0) x [1, T1):
        //   u_A = fma(m_SW, SW_A, fma(m_S, S, fma(m_W, W_A, r0_A))),
        //   u_B = fma(m_SW, W_A, fma(m_S, u_A, fma(m_W, W_B, r0_B)))
        // W from the lane's registers, S = u_B of lane l - 1 by shfl.up (lane 0: row 0), SW = the
        // previous step's S (A) or W_A (B); in place, branch-free (idle lanes of the ramps only
        // predicate their stores and keep their column-0 values)
        if (T0 > 1 && T1 > 1) {
            const int nl = T1 / 2;                                     // lanes with a row
            const int NSTEP = (T0 - 1) + (nl - 1);
            double WA = XN[wi(0, rAl)], WB = XN[wi(0, rBl)], SWA = XN[wi(0, rAl - 1)];
            double uBp = 0.0;
            // the operands of step s (ring coefficients, alpha, r0, row 0) are loaded during step s - 1,
            // ahead of its dependent chain
            auto ldv = [&](int s, double (&c)[6], double &aA, double &aB, double &r0A, double &r0B, double &row0) {
                const int x = s - lane + 1;
                const int xl = x < 1 ? 1 : (x >= T0 ? T0 - 1 : x);
                const double *cr = RING + (s % s9::PD) * s9::RSL + lane;   // [slot][coefficient][lane]
#pragma unroll
                for (int j = 0; j < 6; ++j) c[j] = cr[j * s9::RJL];
                aA = AW[ai(xl, rAl)];
                aB = AW[ai(xl, rBl)];
                r0A = XN[wi(xl, rAl)];
                r0B = XN[wi(xl, rBl)];
                row0 = XN[wi(xl, 0)];
            };
            double c6[6], aA, aB, r0A, r0B, row0;
            const int NC = (NSTEP + CH) / CH;                         // chunks (step NSTEP is read ahead)
            bar_wait(1, bar_cnt(0));                                  // chunk 0 is in the ring
            ldv(0, c6, aA, aB, r0A, r0B, row0);
            for (int s = 0; s < NSTEP; ++s) {
                const int x = s - lane + 1;
                const bool act = onA && x >= 1 && x < T0;
                const int xl = x < 1 ? 1 : (x >= T0 ? T0 - 1 : x);
                const double mWA = aA * c6[0], mSA = aA * c6[1], mDA = aA * c6[2];
                const double mWB = aB * c6[3], mSB = aB * c6[4], mDB = aB * c6[5];
                const double cr0A = r0A, cr0B = r0B, crow0 = row0;
                // step s + 1 opens chunk c + 1: the chunk c this step closes has been read (this step's
                // operands are in registers), its half may be refilled; wait for chunk c + 1
                if ((s + 1) % CH == 0) {
                    const int c = (s + 1) / CH - 1;
                    if (c + 2 < NC) bar_arrive(3 + (c & 1), bar_cnt(c & 1));
                    bar_wait(1 + ((c + 1) & 1), bar_cnt((c + 1) & 1));
                }
                ldv(s + 1, c6, aA, aB, r0A, r0B, row0);
                const double S = sel_f64(lane == 0, crow0, shfl_up1_f64(uBp));
                const double uA = fma(mDA, SWA, fma(mSA, S, fma(mWA, WA, cr0A)));
                const double uB = fma(mDB, WA, fma(mSB, uA, fma(mWB, WB, cr0B)));
                st_shared_if(XN + wi(xl, rAl), uA, act);
                st_shared_if(XN + wi(xl, rBl), uB, act && onB);
                SWA = sel_f64(act, S, SWA);
                WA = sel_f64(act, uA, WA);
                WB = sel_f64(act, uB, WB);
                uBp = uB;
            }
        }
    } else if (T0 > 1 && T1 > 1) {
        const int pt = (int)threadIdx.x - 32;                                   // producer thread index
        // ---- warps 1..7: the wavefront's coefficient ring; the loads of chunk c + 1 are in flight
        //      while the producers wait for the half of chunk c to be free
        const int nl = T1 / 2, NSTEP = (T0 - 1) + (nl - 1);
        const int NC = (NSTEP + CH) / CH;
        constexpr int NP = s9::NPROD, NE = 32 * 6 * CH, NI = (NE + NP - 1) / NP;     // producer threads, items per chunk
        // item k of a producer thread: ring element e = pt + k NP = ((l * 6 + j) * CH + sl), i.e. step
        // c CH + sl of lane l, coefficient j -- the same (l, j, sl) in every chunk, so the row's source
        // pointer (at column x = 0), the column offset and the ring index are set up once
        const double *psrc[NI];
        int pxo[NI], pdst[NI];
        {
#pragma unroll
            for (int k = 0; k < NI; ++k) {
                const int e = pt + k * NP;
                const int sl = e % CH, lj = e / CH, j = lj % 6, l = lj / 6;
                const int r = 2 * l + 1 + (j >= 3), a = j % 3;
                const bool ok = e < NE && r < T1;
                const int64_t i = gidx(G, gxo(0), gyo(ok ? r : 0), 0);
                psrc[k] = !ok ? nullptr
                              : (a == 0 ? (A.f0 ? A.f0 + i + sx : nullptr)
                                        : (a == 1 ? (A.f1 ? A.f1 + i + sy * P0 : nullptr) : fdg + i + sx + sy * P0));
                pxo[k] = ok ? sl - l + 1 : -(1 << 20);                     // x = c CH + pxo (never in range if !ok)
                pdst[k] = sl * s9::RSL + j * s9::RJL + l;                  // + (c % 2) CH RSL
            }
        }
        const int sgx = sx ? -1 : 1;
        auto pload = [&](int c, double (&v)[NI]) {                         // chunk c into registers
#pragma unroll
            for (int k = 0; k < NI; ++k) {
                const int x = c * CH + pxo[k];
                v[k] = (psrc[k] && x >= 1 && x < T0) ? __ldg(psrc[k] + sgx * x) : 1.0;
            }
        };
        auto pstore = [&](int c, const double (&v)[NI]) {                  // registers into half c % 2
            double *const half = RING + (c & 1) * (CH * s9::RSL);
#pragma unroll
            for (int k = 0; k < NI; ++k) {
                const int x = c * CH + pxo[k];
                if (x >= 1 && x < T0) half[pdst[k]] = v[k];
            }
        };
        double pv[NI];
        pload(0, pv);
        for (int c = 0; c < NC; ++c) {
            if (c >= 2) bar_wait(3 + (c & 1), bar_cnt(c & 1));
            pstore(c, pv);
            bar_arrive(1 + (c & 1), bar_cnt(c & 1));
            if (c + 1 < NC) pload(c + 1, pv);
#if SW_S9_AHEAD > 0
            if (c == SW_S9_AHEAD_AT) {
                // look-ahead: the lines of the box SW_S9_AHEAD launches later (window of x_old, b and
                // the coefficient arrays, clamped to the domain) into L2 while this box runs its fronts
                const int64_t nb = (int64_t)blockIdx.x + SW_S9_AHEAD;
                if (nb < (int64_t)gridDim.x) {
                    const int64_t nX0 = (nb % G.nt[0]) * T0 - 2, nY0 = (nb / G.nt[0] + G.toff[1]) * T1 - 2;
                    const int NL = (T0 + 4 + 15) / 16 + 1;
                    for (int e = pt; e < (T1 + 4) * NL * 6; e += NP) {
                        const int a = e % 6, q = e / 6;
                        int64_t gx = nX0 + 16 * (q % NL), gy = nY0 + q / NL;
                        gx = gx < 0 ? 0 : (gx >= G.ng[0] ? G.ng[0] - 1 : gx);
                        gy = gy < 0 ? 0 : (gy >= G.ng[1] ? G.ng[1] - 1 : gy);
                        const double *base =
                            a == 0 ? A.xo : (a == 1 ? A.b : (a == 2 ? A.f0 : (a == 3 ? A.f1 : (a == 4 ? A.dd : A.da))));
                        if (base) asm volatile("prefetch.global.L2 [%0];" ::"l"(base + gidx(G, gx, gy, 0)));
                    }
                }
            }
#endif
        }
    }
    if (fl) atomicOr(A.flag, 1);
    SW_TMARK(t_fronts);
    SW_TADD(3, t_cs, t_fronts);
    SW_TADD(5, 0, 1);
    __syncthreads();
    for (int e = threadIdx.x; e < T0 * T1; e += s9::NT) {
        const int lx = e % T0, ly = e / T0;
        A.xn[gidx(G, gxo(lx), gyo(ly), 0)] = XN[wi(lx, ly)];
    }
}

inline cudaError_t launch_sweep9(const Sweep9Args &A, cudaStream_t s) {
    const size_t sm = sweep9_smem(A.G);
    static size_t attr = 0;
    if (sm > attr) {
        cudaFuncSetAttribute(k_sweep9<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        cudaFuncSetAttribute(k_sweep9<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        attr = sm;
    }
    const unsigned tiles = (unsigned)((int64_t)A.G.nt[0] * A.G.nt[1]);
    if (A.G.T[0] == 64 && A.G.T[1] == 64) k_sweep9<64><<<tiles, s9::NT, sm, s>>>(A);
    else k_sweep9<0><<<tiles, s9::NT, sm, s>>>(A);
    return cudaGetLastError();
}

}  // namespace sw
