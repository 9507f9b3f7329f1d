// tri2t.cuh -- second phase of the transposed (SYMMETRIC-pairing) triangular solve on 64 x 64
// boxes, sm_100a (DESIGN R-C; SURVEY §8(a) a11-a12, §8(c) C-ILU).
//
// The backward factor of the SYMMETRIC pairing solves (D/alpha + A_I^T) z = r0:
//     z_p = r0_p + sum_{q : p implicit for q} alpha_p c_pq z_q .
// Inside a box the q are p's explicit-side (local +x, +y) neighbours, so phase 1 is the
// forward engine (sweep2v.cuh, MODE_TRI) run from the box's far corner with the coupling
// switched off; it is exact for every node except the coupled start-face nodes, which also
// depend on their partners across the face and, through them, on the partner box.  Those are
// recomputed here, in two launches:
//   stage 0: the chains of 2 x 2 pairs along the two start faces, from k = 63 down to 1 (a pair
//            depends on the pair at k+1 and on phase-1 values only);
//   stage 1: the corner set (4 x 4 or 2 x 2), which needs other boxes' stage-0 results.
// One warp per box: all lanes gather the per-pair operands, then lane 0 runs the y-face chain and
// lane 1 the x-face chain.  Same operations and order as the oracle's transposed trisolve.
#pragma once
#include "common.cuh"
#include "sweep2p.cuh"

namespace sw {

struct Tri2tArgs {
    Geo G;
    int base;
    double omega;
    const double *invd;          // 1/D~ (ILU) or null (SSOR: alpha = omega / a_P)
    const double *fx, *fy;       // faces or null (unit)
    const double *src;           // y (phase-1 right-hand side, before the coef scaling)
    double *z;                   // phase-1 result, corrected in place
    double coef;
    int stage;
    int *flag;
};

template <bool FACES>
__global__ void __launch_bounds__(32) k_tri2t(Tri2tArgs A) {
    SW_JITTER_POINT();
    constexpr int T = 64;
    __shared__ double ch[2][11][T];          // per chain, per quantity, per position k
    const Geo &G = A.G;
    const int lane = threadIdx.x;
    const int tx = blockIdx.x % G.nt[0];
    const int ty = blockIdx.x / G.nt[0];
    const int64_t R0 = tx, R1 = ty + G.toff[1];
    const int sx = ((A.base >> 0) & 1) ^ (int)(R0 & 1);
    const int sy = ((A.base >> 1) & 1) ^ (int)(R1 & 1);
    const bool cx = sx ? (R0 < G.ntg[0] - 1) : (R0 > 0);
    const bool cy = sy ? (R1 < G.ntg[1] - 1) : (R1 > 0);
    if (!cx && !cy) return;
    const int64_t P0 = G.P0;
    const int64_t x0 = (int64_t)tx * T + 2, y0 = (int64_t)ty * T + 2;   // padded index of the box's min corner
    const int64_t dxg = sx ? -1 : 1, dyg = sy ? -P0 : P0;              // local +x / +y in the padded arrays
    const int64_t o00 = (y0 + (sy ? T - 1 : 0)) * P0 + (x0 + (sx ? T - 1 : 0));
    auto at = [&](int c, int t) { return o00 + c * dxg + t * dyg; };
    // face of node i toward local +x, -x, +y, -y
    auto fpx = [&](int64_t i) { return FACES ? (sx ? A.fx[i] : A.fx[i + 1]) : 1.0; };
    auto fmx = [&](int64_t i) { return FACES ? (sx ? A.fx[i + 1] : A.fx[i]) : 1.0; };
    auto fpy = [&](int64_t i) { return FACES ? (sy ? A.fy[i] : A.fy[i + P0]) : 1.0; };
    auto fmy = [&](int64_t i) { return FACES ? (sy ? A.fy[i + P0] : A.fy[i]) : 1.0; };
    auto alpha = [&](int64_t i) {
        if (A.invd) return A.invd[i];
        double xl = 1.0, xh = 1.0, yl = 1.0, yh = 1.0;
        if (FACES) { xl = A.fx[i]; xh = A.fx[i + 1]; yl = A.fy[i]; yh = A.fy[i + P0]; }
        return div_rn(A.omega, ((xl + xh) + (yl + yh)) + G.beta);
    };
    const double *z = A.z;
    enum { R0A, R0B, CA, CB, FA, FB, VA, VB, MAB, MBA, INV };

    if (A.stage == 0) {
        // ---- gather: lane handles positions k = lane + 1 and lane + 33 (<= 63) of both chains
        int fl = 0;
        for (int k = lane + 1; k < T; k += 32) {
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) {        // 0: y-face chain (own (k,0)), 1: x-face chain (own (0,k))
                if (cc == 0 ? !cy : !cx) continue;
                const int64_t io = cc ? at(0, k) : at(k, 0);
                const int64_t ip = cc ? io - dxg : io - dyg;           // partner across the face
                const double ao = alpha(io), ap = alpha(ip);
                double co, cp, fo, fp, vo, vp, mop, mpo;
                if (cc == 0) {      // chain along +x (inner term), fixed term along y
                    co = ao * fpx(io); fo = ao * fpy(io); vo = z[io + dyg]; mop = ao * fmy(io);
                    cp = ap * fpx(ip); fp = ap * fmy(ip); vp = z[ip - dyg]; mpo = ap * fpy(ip);
                } else {            // fixed term along x (inner), chain along +y
                    co = ao * fpy(io); fo = ao * fpx(io); vo = z[io + dxg]; mop = ao * fmx(io);
                    cp = ap * fpy(ip); fp = ap * fmx(ip); vp = z[ip - dxg]; mpo = ap * fpx(ip);
                }
                const double r0o = A.coef * A.src[io], r0p = A.coef * A.src[ip];
                const bool pfirst = cc ? (sx == 0) : (sy == 0);          // partner has the lower global index
                double *q = &ch[cc][0][0];
                q[R0A * T + k] = pfirst ? r0p : r0o;
                q[R0B * T + k] = pfirst ? r0o : r0p;
                q[CA * T + k] = pfirst ? cp : co;
                q[CB * T + k] = pfirst ? co : cp;
                q[FA * T + k] = pfirst ? fp : fo;
                q[FB * T + k] = pfirst ? fo : fp;
                q[VA * T + k] = pfirst ? vp : vo;
                q[VB * T + k] = pfirst ? vo : vp;
                const double mab = pfirst ? mpo : mop, mba = pfirst ? mop : mpo;
                q[MAB * T + k] = mab;
                q[MBA * T + k] = mba;
                const double m11 = fma(mba, -mab, 1.0);
                fl |= !(fabs(m11) >= 1e-14);
                q[INV * T + k] = div_rn(1.0, m11);
            }
        }
        if (fl) atomicOr(A.flag, 1);
        __syncwarp();
        // ---- the chains, k = 63 .. 1 (the pair at k depends on the pair at k+1)
        if (lane < 2 && (lane == 0 ? cy : cx)) {
            const int cc = lane;
            const bool pfirst = cc ? (sx == 0) : (sy == 0);
            const double *q = &ch[cc][0][0];
            double pa = 0.0, pb = 0.0;                 // the node beyond the end face is not a dependency
            for (int k = T - 1; k >= 1; --k) {
                double ra, rb;
                if (cc == 0) {
                    ra = fma(q[FA * T + k], q[VA * T + k], fma(q[CA * T + k], pa, q[R0A * T + k]));
                    rb = fma(q[FB * T + k], q[VB * T + k], fma(q[CB * T + k], pb, q[R0B * T + k]));
                } else {
                    ra = fma(q[CA * T + k], pa, fma(q[FA * T + k], q[VA * T + k], q[R0A * T + k]));
                    rb = fma(q[CB * T + k], pb, fma(q[FB * T + k], q[VB * T + k], q[R0B * T + k]));
                }
                pb = fma(q[MBA * T + k], ra, rb) * q[INV * T + k];
                pa = fma(q[MAB * T + k], pb, ra);
                const int64_t io = cc ? at(0, k) : at(k, 0);
                A.z[io] = pfirst ? pb : pa;
            }
        }
        return;
    }

    // ---- stage 1: the corner set (lane 0)
    if (lane != 0) return;
    const int64_t io = at(0, 0), ix = io - dxg, iy = io - dyg, id = io - dxg - dyg;
    // members in ascending global index: (lo y, lo x), (lo y, hi x), (hi y, lo x), (hi y, hi x)
    const int xlo_p = (sx == 0), ylo_p = (sy == 0);
    if (cx && cy) {
        double M[4][4], rhs[4], uu[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            const int isx = (m & 1) ? !xlo_p : xlo_p;
            const int isy = (m & 2) ? !ylo_p : ylo_p;
            const int64_t i = io - (isx ? dxg : 0) - (isy ? dyg : 0);
            const double a = alpha(i);
            // fixed terms: along x then y, toward +x/+y for our-side coordinates, away for partner sides
            const int64_t jx = isx ? i - dxg : i + dxg, jy = isy ? i - dyg : i + dyg;
            const double cxf = a * (isx ? fmx(i) : fpx(i)), cyf = a * (isy ? fmy(i) : fpy(i));
            rhs[m] = fma(cyf, z[jy], fma(cxf, z[jx], A.coef * A.src[i]));
#pragma unroll
            for (int q = 0; q < 4; ++q) M[m][q] = (m == q) ? 1.0 : 0.0;
            M[m][m ^ 1] = -(a * (isx ? fpx(i) : fmx(i)));
            M[m][m ^ 2] = -(a * (isy ? fpy(i) : fmy(i)));
        }
        ge_solve_k<4>(M, rhs, uu, A.flag);
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            const int isx = (m & 1) ? !xlo_p : xlo_p;
            const int isy = (m & 2) ? !ylo_p : ylo_p;
            if (!isx && !isy) A.z[io] = uu[m];
        }
    } else {
        // one coupled face: members own and its partner across that face
        const bool px_ = cx;
        const int64_t ip = px_ ? ix : iy;
        const double ao = alpha(io), ap = alpha(ip);
        // own: fixed terms +x then +y (one of them is the partner side only when coupled, not here)
        const double ro = fma(ao * fpy(io), z[io + dyg], fma(ao * fpx(io), z[io + dxg], A.coef * A.src[io]));
        double rp;
        if (px_)   // x-partner: away along x, +y along y
            rp = fma(ap * fpy(ip), z[ip + dyg], fma(ap * fmx(ip), z[ip - dxg], A.coef * A.src[ip]));
        else       // y-partner: +x along x, away along y
            rp = fma(ap * fmy(ip), z[ip - dyg], fma(ap * fpx(ip), z[ip + dxg], A.coef * A.src[ip]));
        const double mop = ao * (px_ ? fmx(io) : fmy(io)), mpo = ap * (px_ ? fpx(ip) : fpy(ip));
        const bool pfirst = px_ ? xlo_p : ylo_p;
        double M[2][2], rhs[2], uu[2];
        M[0][0] = M[1][1] = 1.0;
        rhs[0] = pfirst ? rp : ro;
        rhs[1] = pfirst ? ro : rp;
        M[0][1] = -(pfirst ? mpo : mop);
        M[1][0] = -(pfirst ? mop : mpo);
        ge_solve_k<2>(M, rhs, uu, A.flag);
        A.z[io] = pfirst ? uu[1] : uu[0];
    }
}

inline cudaError_t launch_tri2t_stage(const Geo &G, int base, double omega, const double *invd, const double *fx,
                                      const double *fy, const double *src, double *z, double coef, int *flag, int stage,
                                      cudaStream_t s) {
    Tri2tArgs A;
    A.G = G;
    A.base = base;
    A.omega = omega;
    A.invd = invd;
    A.fx = fx;
    A.fy = fy;
    A.src = src;
    A.z = z;
    A.coef = coef;
    A.flag = flag;
    A.stage = stage;
    const unsigned tiles = (unsigned)((int64_t)G.nt[0] * G.nt[1]);
    if (fx) k_tri2t<true><<<tiles, 32, 0, s>>>(A);
    else k_tri2t<false><<<tiles, 32, 0, s>>>(A);
    return cudaGetLastError();
}

}  // namespace sw
