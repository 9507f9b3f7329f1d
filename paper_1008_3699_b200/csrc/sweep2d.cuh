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
    CUtensorMap x[2];
    CUtensorMap b;       // 64 x 64 tiles of b (L2 prefetch)
    CUtensorMap f[2];    // 64 x 64 tiles of F_x, F_y (L2 prefetch; variable coefficients only)
    bool ok = false, fok = false;
};

struct Sweep2dArgs {
    Geo G;
    int base;
    double omega[4];
    const double *b;    // padded b
    const double *f0, *f1;   // padded face arrays (FACES)
    double *xnew;       // padded x_new
    int *flag;
};

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
    const double sx = fxb<FACES>(fx, wr, wc - 1) + fxb<FACES>(fx, wr, wc);
    const double sy = fyb<FACES>(fy, wr - 1, wc) + fyb<FACES>(fy, wr, wc);
    return (sx + sy) + beta;
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
__host__ __device__ constexpr size_t sweep2d_smem() {
    // window (r0 in place) + FACES: per-node west/south couplings + y-chain arrays
    return sizeof(double) * (WSZ + (FACES ? 2 * T2 * T2 : 0) + 6 * T2 + 16) + 16;
}

// Explicit part of one node (DESIGN R-7): r0 = fma(alpha, b + c_ex u_ex + c_ey u_ey, (1-w) u_old)
// plus the couplings alpha * c on its two implicit sides.
struct NodeR0 {
    double r0, mx, my;
};

// One box, start corner (SX, SY) known at compile time (bit set = starts at the max end).
template <bool FACES, int SX, int SY>
__device__ __forceinline__ void sweep2d_tile(const CUtensorMap *tmx, const Sweep2dArgs &A, double *sm, uint64_t *bar,
                                             int tx, int ty, bool cx, bool cy) {
    double *xw = sm;                              // x window (global orientation); r0 / results in place
    double *mWt = xw + WSZ;                       // FACES: alpha * c_west per own node, local (c,t) -> [t][c]
    double *mSt = mWt + (FACES ? T2 * T2 : 0);    // FACES: alpha * c_south
    double *ycA = mSt + (FACES ? T2 * T2 : 0);    // y-chain per column c: partner external coupling
    double *ycB = ycA + T2;                       // y-chain: mab
    double *ycC = ycB + T2;                       // y-chain: mba
    double *ycD = ycC + T2;                       // y-chain: 1 / pivot

    const Geo &G = A.G;
    const int lane = threadIdx.x;
    const int x0 = tx * T2;                       // global = local along x
    const int y0l = ty * T2;                      // slab-local
    constexpr int bits = SX | (SY << 1);
    const double beta = G.beta;
    const int64_t P0 = G.P0;
    constexpr int dX = SX ? -1 : 1;               // window word step for local +x
    constexpr int dY = SY ? -WW : WW;             // window word step for local +y
    auto WX = [](int c) { return 2 + (SX ? T2 - 1 - c : c); };
    auto WY = [](int t) { return 2 + (SY ? T2 - 1 - t : t); };
    // padded global index of window word i = wr*WW + wc  (window origin = padded (x0, y0l))
    auto PI = [&](int i) { return (int64_t)(y0l + i / WW) * P0 + (x0 + i % WW); };
    const double *Bg = A.b, *Fx = A.f0, *Fy = A.f1;
    const double w_own = A.omega[bits], w_px = A.omega[bits ^ 1], w_py = A.omega[bits ^ 2];

    // gathered node data (partners, chain constants); faces from global memory
    auto node = [&](int i, int ex, int ey, double w, double bval) {
        NodeR0 o;
        double a0 = 1.0, a1 = 1.0, a2 = 1.0, a3 = 1.0;
        if constexpr (FACES) {
            const int64_t g = PI(i);
            a0 = __ldg(Fx + g);
            a1 = __ldg(Fx + g + 1);
            a2 = __ldg(Fy + g);
            a3 = __ldg(Fy + g + P0);
        }
        const double s = (a0 + a1) + (a2 + a3);     // a_P (R-7), beta added below
        const double al = w / (s + beta);
        const double cex = ex > 0 ? a1 : a0, cey = ey > 0 ? a3 : a2;
        const double cix = ex > 0 ? a0 : a1, ciy = ey > 0 ? a2 : a3;
        double e = fma(cex, xw[i + ex], bval);
        e = fma(cey, xw[i + ey], e);
        o.r0 = fma(al, e, (1.0 - w) * xw[i]);
        o.mx = al * cix;
        o.my = al * ciy;
        return o;
    };

    // ------------------------------------------------------------------ stage-in
    // register ring for the row-streamed b (and faces) of the own-node prologue
    constexpr int RING = FACES ? 8 : 16;
    const int wcl = 2 + 2 * lane;                 // lane's first window column
    const int64_t gcol = x0 + wcl;
    auto grow = [&](int t) { return (int64_t)(y0l + WY(t)) * P0 + gcol; };
    double2 rb[RING], rfx[RING], rfy[RING];
    double rfe[RING];
    auto issue = [&](int t, int slot) {
        const int64_t g = grow(t);
        rb[slot] = __ldg(reinterpret_cast<const double2 *>(Bg + g));
        if constexpr (FACES) {
            rfx[slot] = __ldg(reinterpret_cast<const double2 *>(Fx + g));
            rfe[slot] = (lane == 31) ? __ldg(Fx + g + 2) : 0.0;
            rfy[slot] = __ldg(reinterpret_cast<const double2 *>(Fy + g + (SY ? 0 : P0)));   // explicit-side F_y
        }
    };
#pragma unroll
    for (int t = 0; t < RING; ++t) issue(t, t);
    // partner right-hand sides (independent loads, issued before waiting for the window)
    const int io00 = WY(0) * WW + WX(0);
    double bpx[2] = {0.0, 0.0}, bpy[2] = {0.0, 0.0}, bpd = 0.0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int k = h * 32 + lane;
        if (cx) bpx[h] = __ldg(Bg + PI(WY(k) * WW + WX(0) - dX));
        if (cy) bpy[h] = __ldg(Bg + PI(WY(0) * WW + WX(k) - dY));
    }
    if (cx && cy && lane == 0) bpd = __ldg(Bg + PI(io00 - dX - dY));

    mbar_wait(bar, 0);
    __syncwarp();

    // ------------------------------------------------------------------ prologue: partners
    // (read only halo values; results kept in registers / written after all reads)
    NodeR0 px_[2], py_[2], pd_ = {0.0, 0.0, 0.0};
    double xmab[2] = {0, 0}, xmba[2] = {0, 0}, xinv[2] = {0, 0};
    double ymab[2] = {0, 0}, ymba[2] = {0, 0}, yinv[2] = {0, 0};
    NodeR0 own00 = {0.0, 0.0, 0.0};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int k = h * 32 + lane;          // row t (x-chain) / column c (y-chain)
        px_[h] = {0.0, 0.0, 0.0};
        py_[h] = {0.0, 0.0, 0.0};
        if (cx) {
            const int io = WY(k) * WW + WX(0), ip = io - dX;
            px_[h] = node(ip, -dX, dY, w_px, bpx[h]);          // partner: x flipped, y as ours
            const NodeR0 ow = node(io, dX, dY, w_own, 0.0);    // own couplings
            if (h == 0) own00 = ow;
            const double mop = ow.mx, mpo = px_[h].mx;         // couplings across the shared face
            const double mab = SX ? mop : mpo, mba = SX ? mpo : mop;   // partner first iff SX == 0
            const double M11 = fma(mba, -mab, 1.0);
            if (!(fabs(M11) >= 1e-14)) atomicOr(A.flag, 1);
            xmab[h] = mab;
            xmba[h] = mba;
            xinv[h] = 1.0 / M11;
        }
        if (cy) {
            const int io = WY(0) * WW + WX(k), ip = io - dY;
            py_[h] = node(ip, dX, -dY, w_py, bpy[h]);
            const NodeR0 ow = node(io, dX, dY, w_own, 0.0);
            if (h == 0) own00 = ow;
            const double mop = ow.my, mpo = py_[h].my;
            const double mab = SY ? mop : mpo, mba = SY ? mpo : mop;
            const double M11 = fma(mba, -mab, 1.0);
            if (!(fabs(M11) >= 1e-14)) atomicOr(A.flag, 1);
            ymab[h] = mab;
            ymba[h] = mba;
            yinv[h] = 1.0 / M11;
        }
    }
    if (cx && cy && lane == 0) pd_ = node(io00 - dX - dY, -dX, -dY, A.omega[bits ^ 3], bpd);
    const NodeR0 cpx = px_[0], cpy = py_[0];
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int k = h * 32 + lane;
        if (cy) {
            ycA[k] = py_[h].mx;                 // partner's external (west) coupling
            ycB[k] = ymab[h];
            ycC[k] = ymba[h];
            ycD[k] = yinv[h];
            xw[WY(0) * WW + WX(k) - dY] = py_[h].r0;     // partner r0 in place (row -1)
        }
    }
    __syncwarp();

    // ------------------------------------------------------------------ prologue: own r0
    // Rows in increasing local t (row t reads old row t+1, which the same lane overwrites one
    // iteration later).  Lane l owns window columns 2+2l, 3+2l: 16-byte shared and global
    // accesses, the east value of the neighbouring column via shuffles.
    {
        double2 fyc = make_double2(0.0, 0.0);          // F_y on the implicit side of row t
        if constexpr (FACES) fyc = __ldg(reinterpret_cast<const double2 *>(Fy + grow(0) + (SY ? P0 : 0)));
        const double omw = 1.0 - w_own;
        const double alc = w_own / (4.0 + beta);
        for (int t0 = 0; t0 < T2; t0 += RING) {
#pragma unroll
            for (int k = 0; k < RING; ++k) {
                const int t = t0 + k;
                const int i = WY(t) * WW + wcl;
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
                const double2 bb = rb[k];
                double r00, r01;
                if constexpr (FACES) {
                    const double2 fxv = rfx[k];
                    const double fxr = __shfl_down_sync(0xffffffffu, fxv.x, 1);
                    const double fx2 = (lane == 31) ? rfe[k] : fxr;
                    const double2 fyn = rfy[k];
                    const double xm0 = fxv.x, xp0 = fxv.y, xm1 = fxv.y, xp1 = fx2;
                    const double ym0 = SY ? fyn.x : fyc.x, yp0 = SY ? fyc.x : fyn.x;
                    const double ym1 = SY ? fyn.y : fyc.y, yp1 = SY ? fyc.y : fyn.y;
                    const double s0 = (xm0 + xp0) + (ym0 + yp0), s1 = (xm1 + xp1) + (ym1 + yp1);
                    const double al0 = w_own / (s0 + beta), al1 = w_own / (s1 + beta);
                    double ea = fma(SX ? xm0 : xp0, e0, bb.x);
                    ea = fma(SY ? ym0 : yp0, nb.x, ea);
                    double eb = fma(SX ? xm1 : xp1, e1, bb.y);
                    eb = fma(SY ? ym1 : yp1, nb.y, eb);
                    r00 = fma(al0, ea, (1.0 - w_own) * own.x);
                    r01 = fma(al1, eb, (1.0 - w_own) * own.y);
                    const int c0 = SX ? T2 - 1 - (wcl - 2) : wcl - 2;
                    const int c1 = SX ? c0 - 1 : c0 + 1;
                    mWt[t * T2 + c0] = al0 * (SX ? xp0 : xm0);
                    mSt[t * T2 + c0] = al0 * (SY ? yp0 : ym0);
                    mWt[t * T2 + c1] = al1 * (SX ? xp1 : xm1);
                    mSt[t * T2 + c1] = al1 * (SY ? yp1 : ym1);
                    fyc = fyn;
                } else {
                    double ea = fma(1.0, e0, bb.x);
                    ea = fma(1.0, nb.x, ea);
                    double eb = fma(1.0, e1, bb.y);
                    eb = fma(1.0, nb.y, eb);
                    r00 = fma(alc, ea, omw * own.x);
                    r01 = fma(alc, eb, omw * own.y);
                }
                *reinterpret_cast<double2 *>(xw + i) = make_double2(r00, r01);
                if (t + RING < T2) issue(t + RING, k);
            }
        }
        __syncwarp();
    }

    // ------------------------------------------------------------------ corner (step 0, lane 0)
    double u = 0.0, par = 0.0, Wpy = 0.0, W = 0.0;
    int px = 0;
    if (lane == 0) {
        const int io = io00, ipx = io - dX, ipy = io - dY;
        const double r0o = xw[io];
        if (cx && cy) {
            // members in ascending global index: (low y, low x), (low y, high x), (high y, low x), (high y, high x)
            constexpr int xlo_is_p = (SX == 0), ylo_is_p = (SY == 0);
            double M[4][4], rhs[4], uu[4];
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                const int isx = (m & 1) ? !xlo_is_p : xlo_is_p;
                const int isy = (m & 2) ? !ylo_is_p : ylo_is_p;
                const NodeR0 nd = (isx && isy) ? pd_ : (isx ? cpx : (isy ? cpy : own00));
#pragma unroll
                for (int q = 0; q < 4; ++q) M[m][q] = (m == q) ? 1.0 : 0.0;
                rhs[m] = (isx || isy) ? nd.r0 : r0o;
                M[m][m ^ 1] = -nd.mx;       // towards the member across the x face
                M[m][m ^ 2] = -nd.my;       // towards the member across the y face
            }
            ge_small<4>(M, rhs, uu, A.flag);
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                const int isx = (m & 1) ? !xlo_is_p : xlo_is_p;
                const int isy = (m & 2) ? !ylo_is_p : ylo_is_p;
                xw[io - (isx ? dX : 0) - (isy ? dY : 0)] = uu[m];
                if (!isx && !isy) u = uu[m];
                if (isx && !isy) par = uu[m];
                if (!isx && isy) Wpy = uu[m];
            }
        } else if (cx) {
            const double ro = r0o, rp = cpx.r0;
            const double ra = SX ? ro : rp, rb = SX ? rp : ro;
            const double ub = fma(xmba[0], ra, rb) * xinv[0];
            const double ua = fma(xmab[0], ub, ra) * 1.0;
            u = SX ? ua : ub;
            par = SX ? ub : ua;
            xw[ipx] = par;
        } else if (cy) {
            const double ro = r0o, rp = cpy.r0;
            const double ra = SY ? ro : rp, rb = SY ? rp : ro;
            const double ub = fma(ycC[0], ra, rb) * ycD[0];
            const double ua = fma(ycB[0], ub, ra) * 1.0;
            u = SY ? ua : ub;
            Wpy = SY ? ub : ua;
            xw[ipy] = Wpy;
        } else {
            u = r0o;
        }
        xw[io] = u;
        W = u;
        px = io + dX;
    }
    __syncwarp();

    // ------------------------------------------------------------------ wavefront
    // u(c,t) = fma(mS, S, fma(mW, W, r0)): W = own previous result, S = lane-1's previous result.
    // Coupled pairs (x-face at column 0, y-face on lane 0's row 0) go through one small block.
    const double alc = FACES ? 0.0 : w_own / (4.0 + beta);
    auto step = [&](bool active, int band, int c, bool XCH, bool YCH) {
        const double Ssh = __shfl_up_sync(0xffffffffu, u, 1);
        double Psh = 0.0;
        if (XCH) Psh = __shfl_up_sync(0xffffffffu, par, 1);
        if (active) {
            const int t = band * 32 + lane;
            if (c == 0) {
                px = WY(t) * WW + WX(0);
                W = 0.0;
            }
            const int i = px;
            const double r0 = xw[i];
            double S = Ssh;
            if (lane == 0) S = band ? xw[i - dY] : 0.0;
            double mW = alc, mS = alc;
            if constexpr (FACES) {
                mW = mWt[t * T2 + c];
                mS = mSt[t * T2 + c];
            }
            const double r = fma(mW, W, r0);
            double uu = fma(mS, S, r);
            const bool isx = XCH && (c == 0) && cx;
            const bool isy = YCH && (lane == 0) && (band == 0) && cy;
            if (isx || isy) {
                double ro, rp, mab, mba, inv1;
                bool pfirst;
                if (isx) {      // x-start-face pair of row t: externals are both souths
                    const bool b1 = band != 0;
                    const double Pp = (lane != 0) ? Psh : xw[i - dX - dY];
                    ro = fma(mS, S, r0);
                    rp = fma(b1 ? px_[1].my : px_[0].my, Pp, b1 ? px_[1].r0 : px_[0].r0);
                    mab = b1 ? xmab[1] : xmab[0];
                    mba = b1 ? xmba[1] : xmba[0];
                    inv1 = b1 ? xinv[1] : xinv[0];
                    pfirst = (SX == 0);
                } else {        // y-start-face pair of column c: externals are both wests
                    ro = r;
                    rp = fma(ycA[c], Wpy, xw[i - dY]);
                    mab = ycB[c];
                    mba = ycC[c];
                    inv1 = ycD[c];
                    pfirst = (SY == 0);
                }
                const double ra = pfirst ? rp : ro, rb = pfirst ? ro : rp;
                const double ub = fma(mba, ra, rb) * inv1;
                const double ua = fma(mab, ub, ra) * 1.0;
                uu = pfirst ? ub : ua;
                const double pv = pfirst ? ua : ub;
                if (isx) {
                    par = pv;
                    xw[i - dX] = pv;
                } else {
                    Wpy = pv;
                    xw[i - dY] = pv;
                }
            }
            xw[i] = uu;
            u = uu;
            W = uu;
            px = i + dX;
        }
        __syncwarp();
    };
    for (int s = 1; s < 32; ++s) step(s >= lane, 0, s - lane, true, true);          // A: lanes join
    for (int s = 32; s < 64; ++s) step(true, 0, s - lane, false, true);             // B
    for (int s = 64; s < 96; ++s) {                                                  // C: band switch
        const int k = s - lane;
        step(true, k >> 6, k & 63, true, false);
    }
    for (int s = 96; s < 128; ++s) step(true, 1, s - 64 - lane, false, false);      // D
    for (int s = 128; s < 159; ++s) step(s < 128 + lane, 1, s - 64 - lane, false, false);   // E: lanes leave

    // write back the 64 x 64 interior, one bulk copy per row
    fence_proxy_async_smem();
    __syncwarp();
    for (int rr = lane; rr < T2; rr += 32) {
        double *dst = A.xnew + (int64_t)(y0l + rr + 2) * P0 + (x0 + 2);
        bulk_store(dst, xw + (rr + 2) * WW + 2, T2 * sizeof(double));
    }
    bulk_commit();
    bulk_wait_read0();
}

template <bool FACES>
__global__ void __launch_bounds__(32, FACES ? 2 : 5)
    k_sweep2d(const __grid_constant__ CUtensorMap tmx, Sweep2dArgs A) {
    extern __shared__ __align__(128) double sm[];
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
    }
    __syncwarp();
    if (lane == 0) {
        mbar_expect_tx(&bar, sizeof(double) * WSZ);
        tma_load_2d(sm, &tmx, tx * T2, ty * T2, &bar);
    }
    switch (sx | (sy << 1)) {
        case 0: sweep2d_tile<FACES, 0, 0>(&tmx, A, sm, &bar, tx, ty, cx, cy); break;
        case 1: sweep2d_tile<FACES, 1, 0>(&tmx, A, sm, &bar, tx, ty, cx, cy); break;
        case 2: sweep2d_tile<FACES, 0, 1>(&tmx, A, sm, &bar, tx, ty, cx, cy); break;
        default: sweep2d_tile<FACES, 1, 1>(&tmx, A, sm, &bar, tx, ty, cx, cy); break;
    }
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

inline bool make_maps2d(Maps2d &M, const double *x0, const double *x1, const double *b, const double *fx,
                        const double *fy, int64_t pad0, int64_t pad1) {
    M.ok = encode_2d(&M.x[0], x0, pad0, pad1, WW, WW) && encode_2d(&M.x[1], x1, pad0, pad1, WW, WW) &&
           encode_2d(&M.b, b, pad0, pad1, T2, T2);
    M.fok = fx && fy && encode_2d(&M.f[0], fx, pad0, pad1, T2, T2) && encode_2d(&M.f[1], fy, pad0, pad1, T2, T2);
    return M.ok;
}

inline cudaError_t launch_sweep2d(const Maps2d &M, int cur, const Geo &G, int base, const double *w8,
                                  const double *b, const double *const F[3], double *xn, int *flag, bool faces,
                                  cudaStream_t s) {
    Sweep2dArgs A;
    A.G = G;
    A.base = base;
    for (int i = 0; i < 4; ++i) A.omega[i] = w8[i];
    A.b = b;
    A.f0 = F[0];
    A.f1 = F[1];
    A.xnew = xn;
    A.flag = flag;
    unsigned tiles = (unsigned)((int64_t)G.nt[0] * G.nt[1]);
    if (faces) {
        size_t sm = sweep2d_smem<true>();
        cudaFuncSetAttribute(k_sweep2d<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k_sweep2d<true><<<tiles, 32, sm, s>>>(M.x[cur], A);
    } else {
        size_t sm = sweep2d_smem<false>();
        cudaFuncSetAttribute(k_sweep2d<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k_sweep2d<false><<<tiles, 32, sm, s>>>(M.x[cur], A);
    }
    return cudaGetLastError();
}

}  // namespace sw
