// sweep3s.cuh -- 3D decomposed SOR sweep and block-triangular solves (7-point stencil), streaming
// version for boxes T0 x T1 x T2 with T1 T2 <= 32, T1 + T2 <= 13 and T0 % 4 == 0, sm_100a
// (SURVEY §8(a) a4-a8, a10-a12).
//
// One CTA of two warps per box, no box is ever staged whole:
//  * producer warp P: TMA brings the raw inputs (x_old or the solve's source, b or 1/D~, the
//    three face arrays) in chunks of 4 columns (local x) of a window covering the box, the
//    partner layers across its coupled start faces and their explicit neighbours,
//    into a ring of 3 chunk slots.  From each chunk P forms, row-wise (lanes along x, so every
//    lane does useful work and the addresses are consecutive), the explicit part r0 and the
//    couplings of every node of the box and of its partner layers (DESIGN R-7), and writes them
//    to one small ring per x-line, deep enough for the wavefront's skew; it also factors the
//    4 x 4 sets of the x-edge chain and, before the wavefront, solves the start column (the
//    8 x 8 corner, the y- and z-edge chains, the x-start face pairs).
//  * consumer warp C: lane (j, k) owns the x-line (., j, k) and updates node (s - j - k, j, k)
//    at wavefront step s from its line's ring: the neighbours' new values arrive by shuffles, a
//    node on one coupled face solves its 2 x 2 pair with the partner layer, lane 0 runs the
//    x-edge chain of 4 x 4 sets; results go to a small ring of result chunks that TMA stores.
//  P runs one batch (4 columns) ahead of C, the two meet at a named barrier once per batch.
//  ~50 KB of shared memory per box: four boxes (eight warps) per SM.
// Same operations and order as the oracle (DESIGN R-7, R-8), so the result is bitwise identical.
#pragma once
#include <cuda.h>

#include "common.cuh"
#include "maps2d.cuh"
#include "sweep2p.cuh"
#include "sweep3.cuh"
#include "tma.cuh"

namespace sw {

namespace k3s {
enum { XO = 0, BB = 1, F0 = 2, F1 = 3, F2 = 4 };   // raw inputs: x_old / source, b / 1/D~, faces
}  // namespace k3s

struct Sweep3sArgs {
    Geo G;
    int base;
    double omega[8];
    double coef;
    int *flag;
    int tri, invd_mode, rscale, couple;
    int has_aux;                // the BB window is loaded (b for SOR, 1/D~ for ILU)
    int R[5], Q[5];             // window rows / planes per raw input (host: the TMA boxes)
};

__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, int c0, int c1, int c2, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap *map, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global [%0, {%1, %2, %3}];" ::"l"(map), "r"(c0), "r"(c1), "r"(c2)
                 : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap *map, int c0, int c1, int c2, const void *src) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(map), "r"(c0),
                 "r"(c1), "r"(c2), "r"(smem_u32(src))
                 : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ double shfl_up_w(double v, int d) {
    int lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "d"(v));
    asm volatile("shfl.sync.up.b32 %0, %0, %1, 0, 0xffffffff;" : "+r"(lo) : "r"(d));
    asm volatile("shfl.sync.up.b32 %0, %0, %1, 0, 0xffffffff;" : "+r"(hi) : "r"(d));
    double r;
    asm("mov.b64 %0, {%1, %2};" : "=d"(r) : "r"(lo), "r"(hi));
    return r;
}

// Inputs of one node in local terms: "lo" / "hi" = the face toward local -a / +a, xn[a] the old
// value of the explicit neighbour along a.
struct Raw3 {
    double xo, b, xn[3], flo[3], fhi[3];
};

// r0 and the couplings alpha c toward the implicit sides (DESIGN R-7) of a node whose partner axes
// (local coordinate -1) are L and whose local coordinate is 0 on the axes in lz.  Own nodes take
// the implicit face on local -a and the explicit on local +a; a partner node the reverse along
// its partner axis.  a_P sums each face pair (commutative, so local and global order agree).
template <bool TRI>
__device__ __forceinline__ void node_compact(const Sweep3sArgs &A, const Raw3 &v, int L, int lz, int sb, int cb,
                                             double &r0, double c[3]) {
    const double ap = (((v.flo[0] + v.fhi[0]) + (v.flo[1] + v.fhi[1])) + (v.flo[2] + v.fhi[2])) + A.G.beta;
    double al;
    if (!TRI) {
        const double w = A.omega[sb ^ L];
        al = div_rn(w, ap);
        double ev = v.b;
#pragma unroll
        for (int a = 0; a < 3; ++a) ev = fma(((L >> a) & 1) ? v.flo[a] : v.fhi[a], v.xn[a], ev);
        r0 = fma(al, ev, (1.0 - w) * v.xo);
    } else {
        al = A.invd_mode ? v.b : div_rn(A.omega[0], ap);
        r0 = A.rscale ? al * v.xo : A.coef * v.xo;
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const bool cut = !((L >> a) & 1) && ((lz >> a) & 1) && !((cb >> a) & 1);
        c[a] = cut ? 0.0 : al * (((L >> a) & 1) ? v.fhi[a] : v.flo[a]);
    }
}

// Shared-memory layout (in doubles) derived from the box shape; host and device use the same
// formulas.  Raw windows per array (rows R / planes Q; local index of row 0 / plane 0 for
// sigma = +1 is lmin / pmin, face axes count faces):
//   XO rows [-2, T1], planes [-2, T2]; BB, F0 rows [-1, T1), planes [-1, T2);
//   F1 faces [-1, T1] x planes [-1, T2); F2 rows [-1, T1) x faces [-1, T2].
struct Lay3 {
    int R[5], Q[5], lmin[5], pmin[5], reg[5];
    int slot, ring, nl, rings, nres, ressz, res, xf, mx, mbar, smem;
    unsigned chunk_bytes;
};
namespace k3s {
constexpr int NR = 3;          // raw chunk slots
}
__host__ __device__ inline int lay_round(int n, int a) { return (n + a - 1) / a * a; }
// entries of the ring of x-line (j, k) at skew j + k: the producer writes batch m (columns up to
// 4m) once the consumer has reached barrier B_{m-1} before step 4m - 12, so the consumer may still
// read column 4m - 12 - skew (and prefetch the next one) while it does
constexpr int RING_EXTRA = 13;
__host__ __device__ inline int ring_depth(int j, int k) { return (j > 0 ? j : 0) + (k > 0 ? k : 0) + RING_EXTRA; }
// first entry of line (j, k) (lines ordered by k, then j, both from -1)
__host__ __device__ inline int ring_first(int T1, int j, int k) {
    const int kk = k + 1, jj = j + 1;                        // rows / lines before
    const int rowsum0 = (T1 * (T1 - 1)) / 2 + RING_EXTRA * (T1 + 1);  // a row with max(k, 0) = 0
    const int km = kk >= 2 ? ((kk - 2) * (kk - 1)) / 2 : 0;  // sum of max(k', 0) over k' < k
    const int before_rows = kk * rowsum0 + (T1 + 1) * km;
    const int K5 = (k > 0 ? k : 0) + RING_EXTRA;
    const int jm = jj >= 2 ? ((jj - 2) * (jj - 1)) / 2 : 0;  // sum of max(j', 0) over j' < j
    return before_rows + jj * K5 + jm;
}
__host__ __device__ inline Lay3 lay3(int T1, int T2, bool faces, bool has_aux) {
    using namespace k3s;
    Lay3 L;
    const int R[5] = {T1 + 3, T1 + 1, T1 + 1, T1 + 2, T1 + 1};
    const int Q[5] = {T2 + 3, T2 + 1, T2 + 1, T2 + 1, T2 + 2};
    int off = 0;
    L.chunk_bytes = 0;
    for (int a = 0; a < 5; ++a) {
        L.R[a] = R[a];
        L.Q[a] = Q[a];
        L.lmin[a] = a == 0 ? -2 : -1;
        L.pmin[a] = a == 0 ? -2 : -1;
        L.reg[a] = off;
        const bool used = a == XO || (a == BB && has_aux) || (a >= F0 && faces);
        if (used) {
            off += lay_round(4 * R[a] * Q[a], 16);           // 128-byte aligned TMA destinations
            L.chunk_bytes += 32u * R[a] * Q[a];
        }
    }
    L.slot = off;
    L.ring = NR * off;
    L.nl = (T1 + 1) * (T2 + 1);
    L.rings = 4 * ring_first(T1, -1, T2);                    // total entries x 4 doubles
    L.nres = (T1 + T2 + 2) / 4 + 1 <= 4 ? 4 : 8;
    L.ressz = lay_round(4 * T1 * T2, 16);
    L.res = L.ring + lay_round(L.rings, 16);
    // the start column's compact arrays (MX) share the result ring: they are read right after B_0,
    // the first result is written after B_2
    const int WSm = 2 * (T1 + 1) * (T2 + 1);
    L.mx = L.res;
    L.xf = lay_round(L.res + (L.nres * L.ressz > 4 * WSm + 80 ? L.nres * L.ressz : 4 * WSm + 80), 16);
    L.mbar = 8 * lay_round(L.xf + 16 * 4, 2);                // after the x-edge results of 16 columns
    L.smem = L.mbar + 8 * NR;
    return L;
}

// Compile-time box shapes: SHAPE 1 = 32 x 8 x 4 (config 5), SHAPE 0 = the launch's box.
template <int SHAPE>
struct Box3 {
    __device__ static int t0(const Geo &G) { return G.T[0]; }
    __device__ static int t1(const Geo &G) { return G.T[1]; }
    __device__ static int t2(const Geo &G) { return G.T[2]; }
};
template <>
struct Box3<1> {
    __device__ static constexpr int t0(const Geo &) { return 32; }
    __device__ static constexpr int t1(const Geo &) { return 8; }
    __device__ static constexpr int t2(const Geo &) { return 4; }
};

#ifdef SW_TRACE
#define S3T(v) long long v = sw_clock()
#define S3ACC(acc, a) acc += sw_clock() - (a)
#define S3ADD(ph, v, tid) do { if (threadIdx.x == (tid)) atomicAdd(&sw_trace_sum[ph], (unsigned long long)(v)); } while (0)
#else
#define S3T(v)
#define S3ACC(acc, a)
#define S3ADD(ph, v, tid)
#endif

__device__ __forceinline__ void named_bar(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
    SW_JITTER_POINT();
}
__device__ __forceinline__ void lds2(const double *p, double &a, double &b) {
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(a), "=d"(b) : "r"(smem_u32(p)));
}
__device__ __forceinline__ void lds2u(uint32_t a, double &x, double &y) {
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(a));
}
__device__ __forceinline__ double lds1u(uint32_t a) {
    double x;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(x) : "r"(a));
    return x;
}
__device__ __forceinline__ void sts1u_if(uint32_t a, double v, bool pred) {
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %2, 0;\n @p st.shared.f64 [%0], %1;\n}\n" ::"r"(a), "d"(v), "r"((int)pred)
                 : "memory");
}
__device__ __forceinline__ void sts2(double *p, double a, double b) {
    asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(smem_u32(p)), "d"(a), "d"(b) : "memory");
}

template <bool FACES, bool TRI, int SHAPE>
__global__ void __launch_bounds__(128, 4)
    k_sweep3s(const __grid_constant__ Sweep3sArgs A, const __grid_constant__ CUtensorMap mXO,
              const __grid_constant__ CUtensorMap mBB, const __grid_constant__ CUtensorMap mF0,
              const __grid_constant__ CUtensorMap mF1, const __grid_constant__ CUtensorMap mF2,
              const __grid_constant__ CUtensorMap mOUT) {
    using namespace k3s;
    extern __shared__ __align__(1024) double sm[];
    SW_JITTER_POINT();
    const Geo &G = A.G;
    using BX = Box3<SHAPE>;
    const int T0 = BX::t0(G), T1 = BX::t1(G), T2 = BX::t2(G);
    const Lay3 Y = lay3(T1, T2, FACES, A.has_aux);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double *const ring = sm;
    // the x-lines' compact rings, entry E = (r0, c0 | c1, c2) split into two arrays of 16-byte halves
    // (rng[2E..] and rng[HB + 2E..]): the wavefront's 16-byte loads of one half then spread over all
    // eight 16-byte bank groups instead of every other one
    double *const rng = sm + Y.ring;
    const int HB = Y.rings / 2;                               // doubles before the second halves
    double *const res = sm + Y.res;
    double *const XE = sm + Y.xf;                             // x-edge results: (u, across z, across y) per column
    double *const MX = sm + Y.mx;
    uint64_t *const bar = reinterpret_cast<uint64_t *>(reinterpret_cast<char *>(sm) + Y.mbar);

    // box, start bits, coupled start faces
    const int tx = blockIdx.x % G.nt[0];
    const int ty = (blockIdx.x / G.nt[0]) % G.nt[1];
    const int tz = blockIdx.x / (G.nt[0] * G.nt[1]);
    const int64_t Rg[3] = {tx, ty, tz + G.toff[2]};
    int sb = 0, cb = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const int s = ((A.base >> a) & 1) ^ (int)(Rg[a] & 1);
        const bool c = A.couple && (s ? (Rg[a] < G.ntg[a] - 1) : (Rg[a] > 0));
        sb |= s << a;
        cb |= (int)c << a;
    }
    const int sx = sb & 1, sy = (sb >> 1) & 1, sz = (sb >> 2) & 1;
    const int X0 = tx * T0, Y0 = ty * T1, Z0 = tz * T2;      // padded coordinates of (box min - 2)
    const int NCH = T0 / 4 + 1;                              // raw chunks = production batches
    // barriers B_1 .. B_MLAST after B_0: the producer forms batch m before B_m, the x-edge warp
    // solves the sets of batch m between B_m and B_{m+1}, the wavefront runs steps [4m - 8, 4m - 4)
    // between B_m and B_{m+1}
    const int MLAST = (T0 + T1 + T2 - 3) / 4 + 2;
    const int RSm = 2, PSm = 2 * (T1 + 1), WSm = PSm * (T2 + 1);
    auto wofm = [&](int l0, int l1, int l2) { return (l0 + 1) + RSm * (l1 + 1) + PSm * (l2 + 1); };
    const int nl = T1 * T2;
    int fl = 0;                                              // singular-pivot flag of this lane

    S3T(t_start);
    if (warp == 1 || warp == 3) {
        // ============================================================ producers
        // warp 1 (pw = 0) also stages the raw chunks (TMA) and solves the start column; the two
        // producer warps form the even / odd rounds of every batch
        const int pw = warp == 3;
        auto org = [&](int arr, int axis) -> int {           // padded global origin of a window axis
            const int lmn = axis == 1 ? Y.lmin[arr] : Y.pmin[arr];
            const int n = axis == 1 ? Y.R[arr] : Y.Q[arr];
            const int T = axis == 1 ? T1 : T2, B0 = axis == 1 ? Y0 : Z0;
            const int fax = (arr == F1 && axis == 1) || (arr == F2 && axis == 2);
            const int rev = axis == 1 ? sy : sz;
            return rev ? B0 + 1 + T - (lmn + n - 1) + fax : B0 + 2 + lmn;
        };
        int oy[5], oz[5];
#pragma unroll
        for (int a = 0; a < 5; ++a) {
            oy[a] = org(a, 1);
            oz[a] = org(a, 2);
        }
        auto chunk_x = [&](int m) { return sx ? X0 + T0 - 4 * m : X0 + 4 * m; };
        auto issue = [&](int m) {                            // lane 0
            const int q = m % NR;
            double *dst = ring + q * Y.slot;
            const int gx = chunk_x(m);
            mbar_expect_tx(&bar[q], Y.chunk_bytes);
            tma_load_3d(dst + Y.reg[XO], &mXO, gx, oy[XO], oz[XO], &bar[q]);
            if (A.has_aux) tma_load_3d(dst + Y.reg[BB], &mBB, gx, oy[BB], oz[BB], &bar[q]);
            if (FACES) {
                tma_load_3d(dst + Y.reg[F0], &mF0, gx, oy[F0], oz[F0], &bar[q]);
                tma_load_3d(dst + Y.reg[F1], &mF1, gx, oy[F1], oz[F1], &bar[q]);
                tma_load_3d(dst + Y.reg[F2], &mF2, gx, oy[F2], oz[F2], &bar[q]);
            }
        };
        auto prefetch = [&](int m) {
            const int gx = chunk_x(m);
            tma_prefetch_3d(&mXO, gx, oy[XO], oz[XO]);
            if (A.has_aux) tma_prefetch_3d(&mBB, gx, oy[BB], oz[BB]);
            if (FACES) {
                tma_prefetch_3d(&mF0, gx, oy[F0], oz[F0]);
                tma_prefetch_3d(&mF1, gx, oy[F1], oz[F1]);
                tma_prefetch_3d(&mF2, gx, oy[F2], oz[F2]);
            }
        };
        auto wait_chunk = [&](int m) { mbar_wait(&bar[m % NR], (m / NR) & 1); };
        if (pw == 0 && lane == 0) {
            for (int q = 0; q < NR; ++q) mbar_init(&bar[q], 1);
            fence_mbar_init();
            for (int m = 0; m < min(NCH, NR); ++m) issue(m);
            for (int m = NR; m < min(NCH, NR + 2); ++m) prefetch(m);
        }
        __syncwarp();
        // word of local column c in the ring (chunk m = columns [4m-2, 4m+2) in slot m % NR)
        auto colw = [&](int col) {
            col = min(max(col, -2), T0 + 1);
            const int m = (col + 2) >> 2;
            const int xs = sx ? 3 - ((col + 2) & 3) : ((col + 2) & 3);
            return (m % NR) * Y.slot + xs;
        };
        auto rho = [&](int arr, int row) { return sy ? (Y.lmin[arr] + Y.R[arr] - 1 - row) : (row - Y.lmin[arr]); };
        auto pio = [&](int arr, int pl) { return sz ? (Y.pmin[arr] + Y.Q[arr] - 1 - pl) : (pl - Y.pmin[arr]); };
        auto rowk = [&](int arr, int row, int pl) { return Y.reg[arr] + 4 * (pio(arr, pl) * Y.R[arr] + rho(arr, row)); };
        // r0 and couplings of node (c, j, k) with partner axes L from the raw ring; wc / wm / wp
        // are the column words of c, c - 1, c + 1
        auto compact = [&](int c, int j, int k, int L, int wc, int wm, int wp, double &r0, double cc[3]) {
            Raw3 v;
            const int kx = rowk(XO, j, k);
            const int dy = sy ? -4 : 4, dzx = (sz ? -4 : 4) * Y.R[XO];
            v.xo = ring[wc + kx];
            v.b = A.has_aux ? ring[wc + rowk(BB, j, k)] : 0.0;
            if (!TRI) {
                v.xn[0] = ring[((L & 1) ? wm : wp) + kx];
                v.xn[1] = ring[wc + kx + ((L & 2) ? -dy : dy)];
                v.xn[2] = ring[wc + kx + ((L & 4) ? -dzx : dzx)];
            } else {
                v.xn[0] = v.xn[1] = v.xn[2] = 0.0;
            }
            if (FACES) {
                const int k0 = rowk(F0, j, k), k1 = rowk(F1, j, k), k2 = rowk(F2, j, k);
                v.flo[0] = ring[(sx ? wm : wc) + k0];        // F_x at node g is the face (g - e_x, g)
                v.fhi[0] = ring[(sx ? wc : wp) + k0];
                v.flo[1] = ring[wc + k1];
                v.fhi[1] = ring[wc + k1 + dy];
                v.flo[2] = ring[wc + k2];
                v.fhi[2] = ring[wc + k2 + (sz ? -4 : 4) * Y.R[F2]];
            } else {
#pragma unroll
                for (int a = 0; a < 3; ++a) v.flo[a] = v.fhi[a] = 1.0;
            }
            const int lz = (c == 0 ? 1 : 0) | (j == 0 ? 2 : 0) | (k == 0 ? 4 : 0);
            node_compact<TRI>(A, v, L, lz, sb, cb, r0, cc);
        };

#ifdef SW_TRACE
        long long t_sets_out = 0;
#endif
        if (pw == 0) {
        // ---- 1. the start column: compact arrays over local columns {-1, 0}, rows [-1, T1),
        //      planes [-1, T2) (X: r0, then the solved values; C0..C2), solved in place
        wait_chunk(0);
        S3T(t_c0);
        S3ADD(0, t_c0 - t_start, 32);
        for (int e = lane; e < WSm; e += 32) {
            const int l0 = e % 2 - 1, l1 = (e / 2) % (T1 + 1) - 1, l2 = e / PSm - 1;
            const int L = (l0 < 0 ? 1 : 0) | (l1 < 0 ? 2 : 0) | (l2 < 0 ? 4 : 0);
            double r0 = 0.0, c[3] = {0.0, 0.0, 0.0};
            if ((L & cb) == L) compact(l0, l1, l2, L, colw(l0), colw(l0 - 1), colw(l0 + 1), r0, c);
            MX[e] = r0;
            MX[WSm + e] = c[0];
            MX[2 * WSm + e] = c[1];
            MX[3 * WSm + e] = c[2];
        }
        __syncwarp();
        S3T(t_mx);
        S3ADD(1, t_mx - t_c0, 32);
        const int stm[3] = {1, RSm, PSm};
        if (__popc(cb) >= 2) {
            if (cb == 7) {
                corner8_coop(MX, WSm, MX + 4 * WSm, lane, wofm(0, 0, 0), stm, sb, A.flag);
            } else {
                if (lane == 0) {
                    const int w = wofm(0, 0, 0);
                    switch (cb) {
                        case 3: solve_set3<3>(MX, WSm, w, stm, sb, A.flag); break;
                        case 5: solve_set3<5>(MX, WSm, w, stm, sb, A.flag); break;
                        default: solve_set3<6>(MX, WSm, w, stm, sb, A.flag); break;
                    }
                }
                __syncwarp();
            }
            // y-edge chain (sets on the x and z faces along y: lanes 0..T1-2) and z-edge chain (x
            // and y faces along z: lanes 16..16+T2-2), factored in parallel, substituted in order
            const bool ych = (cb & 5) == 5, zch = (cb & 3) == 3;
            Fac4 F;
            const bool ymine = ych && lane < 16 && lane + 1 < T1;
            const bool zmine = zch && lane >= 16 && lane - 16 + 1 < T2;
            if (ymine) factor4<5>(MX, WSm, wofm(0, lane + 1, 0), stm, sb, F, fl);
            if (zmine) factor4<3>(MX, WSm, wofm(0, 0, lane - 16 + 1), stm, sb, F, fl);
            const int tmax = max(ych ? T1 : 1, zch ? T2 : 1);
            for (int t = 1; t < tmax; ++t) {
                if (ymine && lane == t - 1) subst4<5>(MX, WSm, wofm(0, t, 0), stm, sb, F);
                if (zmine && lane - 16 == t - 1) subst4<3>(MX, WSm, wofm(0, 0, t), stm, sb, F);
                __syncwarp();
            }
        }
        S3T(t_sets);
        S3ADD(2, t_sets - t_mx, 32);
#ifdef SW_TRACE
        t_sets_out = t_sets;
#endif
        // the x-start face pairs (0, j, k) / (-1, j, k), a 2D recurrence over d = j + k
        if (cb & 1) {
            const bool on = lane < nl;
            const int j = on ? lane % T1 : 0, k = on ? lane / T1 : 0;
            const int m0 = 1 | (j == 0 ? (cb & 2) : 0) | (k == 0 ? (cb & 4) : 0);
            const int w = wofm(0, j, k), q = w - 1;
            const bool qf = sx == 0;
            for (int d = 0; d <= T1 + T2 - 2; ++d) {
                if (on && j + k == d && m0 == 1) {
                    const double rp = fma(MX[3 * WSm + w], MX[w - PSm], fma(MX[2 * WSm + w], MX[w - RSm], MX[w]));
                    const double rq = fma(MX[3 * WSm + q], MX[q - PSm], fma(MX[2 * WSm + q], MX[q - RSm], MX[q]));
                    const double ra = qf ? rq : rp, rb = qf ? rp : rq;
                    const double cw = MX[WSm + w], cq = MX[WSm + q];
                    const double mab = qf ? cq : cw, mba = qf ? cw : cq;
                    const double m11 = fma(mba, -mab, 1.0);
                    fl |= !(fabs(m11) >= 1e-14);
                    const double ub = fma(mba, ra, rb) * div_rn(1.0, m11);
                    const double ua = fma(mab, ub, ra);
                    MX[w] = qf ? ub : ua;
                    MX[q] = qf ? ua : ub;
                }
                __syncwarp();
            }
        }

        }
        // ---- 2. production batches: batch 0 = column 0, batch m >= 1 = columns [4m-3, 4m+1);
        //      lanes: column cs + (lane & 3) of x-line 8 r + (lane >> 2), round r.  Everything but
        //      the column is the same in every batch: per-round word offsets, ring line, depth.
        const int NLn = Y.nl;
        constexpr int MAXR = 4;                               // rounds per producer warp (x-lines / 16)
        const int nr = (NLn + 7) / 8;                         // rounds of both warps (r = 2 i + pw)
        struct PRound {
            int kx, kxy, kxz, kb, k0, k1i, k1e, k2i, k2e, rb, D, pos, L;
            bool on, cuty, cutz;
        };
        PRound pr[MAXR];
        {
            const int dy = sy ? -4 : 4;
#pragma unroll
            for (int i = 0; i < MAXR; ++i) {
                const int r = 2 * i + pw;
                if (r < nr) {
                    const int li = 8 * r + (lane >> 2);
                    const int j = li % (T1 + 1) - 1, k = li / (T1 + 1) - 1;
                    const int L = (j < 0 ? 2 : 0) | (k < 0 ? 4 : 0);
                    PRound &q = pr[i];
                    q.L = L;
                    q.on = li < NLn && (L & cb) == L;
                    q.kx = rowk(XO, j, k);
                    q.kxy = rowk(XO, (L & 2) ? j - 1 : j + 1, k);
                    q.kxz = rowk(XO, j, (L & 4) ? k - 1 : k + 1);
                    q.kb = rowk(BB, j, k);
                    q.k0 = rowk(F0, j, k);
                    const int f1lo = rowk(F1, j, k), f2lo = rowk(F2, j, k);
                    const int f1hi = f1lo + dy, f2hi = f2lo + (sz ? -4 : 4) * Y.R[F2];
                    q.k1i = (L & 2) ? f1hi : f1lo;                     // implicit side: local -a, a partner's +a
                    q.k1e = (L & 2) ? f1lo : f1hi;
                    q.k2i = (L & 4) ? f2hi : f2lo;
                    q.k2e = (L & 4) ? f2lo : f2hi;
                    q.cuty = !(L & 2) && j == 0 && !(cb & 2);
                    q.cutz = !(L & 4) && k == 0 && !(cb & 4);
                    q.rb = 4 * ring_first(T1, j < T1 ? j : 0, k < T2 ? k : 0);
                    q.D = ring_depth(j, k);
                    q.pos = 1 + (lane & 3);                         // ring position of batch 1's column
                }
            }
        }
        auto produce0 = [&]() {                              // batch 0: column 0 (generic path)
            const int c = 0;
            for (int r = 0; 8 * r < NLn; ++r) {
                const int li = 8 * r + (lane >> 2);
                const int j = li % (T1 + 1) - 1, k = li / (T1 + 1) - 1;
                const int L = (j < 0 ? 2 : 0) | (k < 0 ? 4 : 0);
                if ((lane & 3) == 0 && li < NLn && (L & cb) == L) {
                    double r0, cc[3];
                    compact(c, j, k, L, colw(c), colw(c - 1), colw(c + 1), r0, cc);
                    double *e = rng + 2 * ring_first(T1, j, k);
                    sts2(e, r0, cc[0]);
                    sts2(e + HB, cc[1], cc[2]);
                }
            }
        };
        auto produce = [&](int m) {                          // batch m >= 1 (branch-free rounds)
            const int c = 4 * m - 3 + (lane & 3);
            const bool cact = c < T0;
            const int wc = colw(c), wp = colw(c + 1), wm = colw(c - 1);
            const int f0i = sx ? wm : wc, f0e = sx ? wc : wp;
#pragma unroll
            for (int i = 0; i < MAXR; ++i) {
                if (2 * i + pw < nr) {
                    PRound &q = pr[i];
                    const double xo = ring[wc + q.kx];
                    const double b = A.has_aux ? ring[wc + q.kb] : 0.0;
                    double fi0 = 1.0, fe0 = 1.0, fi1 = 1.0, fe1 = 1.0, fi2 = 1.0, fe2 = 1.0;
                    if (FACES) {
                        fi0 = ring[f0i + q.k0];
                        fe0 = ring[f0e + q.k0];
                        fi1 = ring[wc + q.k1i];
                        fe1 = ring[wc + q.k1e];
                        fi2 = ring[wc + q.k2i];
                        fe2 = ring[wc + q.k2e];
                    }
                    const double ap = (((fi0 + fe0) + (fi1 + fe1)) + (fi2 + fe2)) + G.beta;
                    double al, r0;
                    if (!TRI) {
                        const double xnx = ring[wp + q.kx], xny = ring[wc + q.kxy], xnz = ring[wc + q.kxz];
                        const double w = A.omega[sb ^ q.L];
                        al = div_rn(w, ap);
                        r0 = fma(al, fma(fe2, xnz, fma(fe1, xny, fma(fe0, xnx, b))), (1.0 - w) * xo);
                    } else {
                        al = A.invd_mode ? b : div_rn(A.omega[0], ap);
                        r0 = A.rscale ? al * xo : A.coef * xo;
                    }
                    const double c1 = al * fi1, c2 = al * fi2;
                    const uint32_t e = smem_u32(rng + q.rb / 2 + 2 * q.pos);
                    const int on = q.on && cact;
                    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %0, 0;\n"
                                 " @p st.shared.v2.f64 [%1], {%2, %3};\n @p st.shared.v2.f64 [%6], {%4, %5};\n}\n"
                                 ::"r"(on), "r"(e), "d"(r0), "d"(al * fi0), "d"(q.cuty ? 0.0 : c1), "d"(q.cutz ? 0.0 : c2),
                                 "r"(e + 8u * (uint32_t)HB)
                                 : "memory");
                    q.pos += 4;
                    if (q.pos >= q.D) q.pos -= q.D;
                }
            }
        };
        S3T(t_xs);
        S3ADD(3, t_xs - t_sets_out, 32);
        if (pw == 0) produce0();
        __syncwarp();
        named_bar(1, 128);                                    // B_0: start column and batch 0
        S3T(t_b0);
        S3ADD(4, t_b0 - t_xs, 32);
#ifdef SW_TRACE
        long long wch = 0, wbar = 0, p1b2 = 0, p2b2 = 0;
#endif
        for (int m = 1; m < NCH; ++m) {
            S3T(t_w);
            wait_chunk(m);
            S3ACC(wch, t_w);
            produce(m);
            __syncwarp();
            S3T(t_b2);
            named_bar(2, 64);                                // both producers are done with chunk m - 1
#ifdef SW_TRACE
            if (pw) p2b2 += sw_clock() - t_b2; else p1b2 += sw_clock() - t_b2;
#endif
            if (pw == 0 && lane == 0 && m + 2 < NCH) {       // chunk m - 1 is dead: its slot takes m + 2
                fence_proxy_async_smem();
                issue(m + 2);
                if (m + 4 < NCH) prefetch(m + 4);
            }
            __syncwarp();
            S3T(t_bb);
            named_bar(1, 128);                                // B_m
            S3ACC(wbar, t_bb);
        }
        for (int m = NCH; m <= MLAST; ++m) named_bar(1, 128);
#ifdef SW_TRACE
        S3ADD(6, wch, 32);
        S3ADD(14, p1b2, 32);
        S3ADD(15, p2b2, 96);
        S3ADD(7, wbar, 32);
        S3ADD(8, sw_clock() - t_start, 32);
#endif
    } else if (warp == 2) {
        // ============================================================ x-edge chain (warp X)
        // The sets of the y- and z-start faces' common edge along x (members: own line (0, 0),
        // across y (-1, 0), across z (0, -1), both (-1, -1)), one per column c >= 1, each reading
        // the previous column's solution: a serial chain that needs nothing the wavefront computes,
        // so lane 0 runs it one batch ahead of the wavefront.  Members in rank order S = r ^ mm
        // (bit 0 across y, bit 1 across z), factored and substituted exactly as ge_solve_k<4> (the
        // oracle's elimination order, DESIGN R-8).  XE[c % 16] = (u(c,0,0), u(c,0,-1), u(c,-1,0)).
        const bool xe_box = (cb & 6) == 6;
        const int mm = (sy ? 0 : 1) | (sz ? 0 : 2);
        named_bar(1, 128);                                    // B_0
        double er[4] = {0.0, 0.0, 0.0, 0.0};                 // previous set, rank order
        if (xe_box) {
            const double u0 = MX[wofm(0, 0, 0)], py = MX[wofm(0, -1, 0)], pz = MX[wofm(0, 0, -1)];
            const double pyz = MX[wofm(0, -1, -1)];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int S = r ^ mm;
                er[r] = S == 0 ? u0 : (S == 1 ? py : (S == 2 ? pz : pyz));
            }
        }
#ifdef SW_TRACE
        long long xbusy = 0;
#endif
        for (int m = 1; m <= MLAST; ++m) {
            S3T(t_xb);
            const int bt = m - 1;                            // the batch of this interval
            if (xe_box && bt >= 1 && bt < NCH) {
                // lane t < 4 factors the set of the batch's column 4 bt - 3 + t (independent of the
                // chain): multipliers l, eliminated upper triangle U, reciprocal pivots, the rows' r0
                // and x couplings, in registers; then the chain passes from lane to lane: in round t
                // lane t substitutes its set with the previous set's solution, broadcast by shuffles
                const int c = 4 * bt - 3 + lane;
                const bool mine = lane < 4 && c >= 1 && c < T0;
                double fL[6], fU[6], fI[4], fR[4], fX[4];
                {
                    const int pos = (mine ? c : 1) % RING_EXTRA;  // members have skew 0
                    double M[4][4];
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        const int S = r ^ mm, jj = -(S & 1), kk = -(S >> 1);
                        const double *e = rng + 2 * (ring_first(T1, jj, kk) + pos);
#pragma unroll
                        for (int q = 0; q < 4; ++q) M[r][q] = (r == q) ? 1.0 : 0.0;
                        M[r][r ^ 1] = -e[HB];                    // toward the partner across y
                        M[r][r ^ 2] = -e[HB + 1];                // across z
                        fR[r] = e[0];
                        fX[r] = e[1];
                    }
                    int li = 0;
#pragma unroll
                    for (int p = 0; p < 4; ++p) {
                        const double piv = M[p][p];
                        fl |= mine && !(fabs(piv) >= 1e-14);
                        fI[p] = div_rn(1.0, piv);
#pragma unroll
                        for (int q = p + 1; q < 4; ++q) {
                            const double l = M[q][p] * fI[p];
                            fL[li++] = l;
#pragma unroll
                            for (int jj = p + 1; jj < 4; ++jj) M[q][jj] = fma(-l, M[p][jj], M[q][jj]);
                        }
                    }
                    int ui = 0;
#pragma unroll
                    for (int p = 0; p < 4; ++p)
#pragma unroll
                        for (int jj = p + 1; jj < 4; ++jj) fU[ui++] = M[p][jj];
                }
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    // the same operations and order as ge_solve_k<4> (every lane runs them on its own
                    // factors; lane t's result is the chain's)
                    double rhs[4], uu[4];
#pragma unroll
                    for (int r = 0; r < 4; ++r) rhs[r] = fma(fX[r], er[r], fR[r]);
                    int li = 0;
#pragma unroll
                    for (int p = 0; p < 4; ++p)
#pragma unroll
                        for (int q = p + 1; q < 4; ++q) {
                            rhs[q] = fma(-fL[li], rhs[p], rhs[q]);
                            ++li;
                        }
                    constexpr int UI[4] = {0, 3, 5, 6};
#pragma unroll
                    for (int p = 3; p >= 0; --p) {
                        double sacc = rhs[p];
#pragma unroll
                        for (int q = p + 1; q < 4; ++q) sacc = fma(-fU[UI[p] + (q - p - 1)], uu[q], sacc);
                        uu[p] = sacc * fI[p];
                    }
                    const int cc = 4 * bt - 3 + t;
                    if (cc >= 1 && cc < T0) {
#pragma unroll
                        for (int r = 0; r < 4; ++r) er[r] = __shfl_sync(0xffffffffu, uu[r], t);
                        if (lane == 0) {
                            auto pick = [&](int r) { return r == 0 ? er[0] : (r == 1 ? er[1] : (r == 2 ? er[2] : er[3])); };
                            double *w = XE + 4 * (cc & 15);
                            w[0] = pick(mm);
                            w[1] = pick(2 ^ mm);
                            w[2] = pick(1 ^ mm);
                        }
                    }
                }
            }
            __syncwarp();
            S3ACC(xbusy, t_xb);
            named_bar(1, 128);                                // B_m
        }
        S3ADD(13, xbusy, 64);
    } else {
        // ============================================================ consumer
        const bool onl = lane < nl;
        const int j = onl ? lane % T1 : 0, k = onl ? lane / T1 : 0;
        const int m0 = (cb & 1) | (j == 0 ? (cb & 2) : 0) | (k == 0 ? (cb & 4) : 0);   // coupled axes at c = 0
        const int m1 = (j == 0 ? (cb & 2) : 0) | (k == 0 ? (cb & 4) : 0);              // and at c >= 1
        const bool set0 = onl && __popc(m0) >= 2;
        const bool pre0 = onl && ((cb & 1) || set0);        // node (0, j, k) solved by the producer
        const bool xedge = onl && m1 == 6;                   // lane 0: x-edge chain
        const bool xe_box = (cb & 6) == 6;
        const int pax = (m1 == 2) ? 1 : (m1 == 4 ? 2 : -1); // pair axis at c >= 1
        const int pj = pax == 1 ? -1 : j, pk = pax == 2 ? -1 : k;
        const int qf = pax < 0 ? 1 : (((sb >> pax) & 1) == 0);
        const int Do = ring_depth(j, k), Dp = ring_depth(pj, pk);
        const double *const ro = rng + 2 * ring_first(T1, j, k);
        const double *const rp_ = rng + 2 * ring_first(T1, pj, pk);
        const int rrow = ((sz ? T2 - 1 - k : k) * T1 + (sy ? T1 - 1 - j : j)) * 4;
        named_bar(1, 128);                                    // B_0
        S3T(t_cb0);
        S3ADD(9, t_cb0 - t_start, 0);
        S3ADD(5, 1, 0);
#ifdef SW_TRACE
        long long cbar = 0;
#endif
        double u0 = 0.0, sS0 = 0.0, sB0 = 0.0, wq0 = 0.0;
        if (pre0) {
            u0 = MX[wofm(0, j, k)];
            const double px = (m0 & 1) ? MX[wofm(-1, j, k)] : 0.0;
            sS0 = sB0 = px;
            if (j == 0 && k == 0) {
                const double py = (cb & 2) ? MX[wofm(0, -1, 0)] : 0.0, pz = (cb & 4) ? MX[wofm(0, 0, -1)] : 0.0;
                if (!(cb & 1)) {
                    sS0 = pz;
                    sB0 = py;
                }
            }
            if (m1 == 2) wq0 = MX[wofm(0, -1, k)];
            if (m1 == 4) wq0 = MX[wofm(0, j, -1)];
        }
        const int NS = T0 + T1 + T2 - 2, lag = T1 + T2 - 2, NQ = T0 / 4;
        int c = -j - k, po = 0, pp = 0;                      // column; ring positions of column c
        double W = 0.0, Wq = 0.0, u = 0.0, sS = 0.0, sB = 0.0;
        // 32-bit shared addresses (no generic-to-shared conversion in the loop)
        const uint32_t ro_a = smem_u32(ro), rp_a = smem_u32(rp_), xe_a = smem_u32(XE);
        const uint32_t hb_b = 8u * (uint32_t)HB;             // byte offset of the second halves
        const uint32_t res_a = smem_u32(res) + 8 * (rrow);
        // coefficients of the step's column, prepared a step ahead (off the wavefront's dependence
        // chain): the couplings without the pair axis, the pair couplings and 1 / (1 - m m')
        struct Co {
            double r0, c0, e1, e2, q0, d0, f1, f2, mab, mba, inv;
            bool sing;
        };
        auto prep = [&](Co &o) {
            double c1, c2, d1, d2;
            lds2u(ro_a + 16 * po, o.r0, o.c0);
            lds2u(ro_a + 16 * po + hb_b, c1, c2);
            lds2u(rp_a + 16 * pp, o.q0, o.d0);
            lds2u(rp_a + 16 * pp + hb_b, d1, d2);
            const double cpp = pax == 1 ? c1 : c2, cqp = pax == 1 ? d1 : d2;
            o.e1 = pax == 1 ? 0.0 : c1;
            o.e2 = pax == 2 ? 0.0 : c2;
            o.f1 = pax == 1 ? 0.0 : d1;
            o.f2 = pax == 2 ? 0.0 : d2;
            o.mab = pax < 0 ? 0.0 : (qf ? cqp : cpp);
            o.mba = pax < 0 ? 0.0 : (qf ? cpp : cqp);
            const double m11 = fma(o.mba, -o.mab, 1.0);
            o.sing = pax >= 0 && !(fabs(m11) >= 1e-14);
            o.inv = div_rn(1.0, m11);
        };
        Co co;
        prep(co);                                            // (entries of column c < 0: never used)
        int passed = 0;                                      // barriers passed after B_0
#pragma unroll 1
        for (int s = 0; s < NS; ++s, ++c) {
            if ((s & 3) == 0) {                              // steps [4m - 8, 4m - 4) run after B_m
                S3T(t_cb);
                while (passed < s / 4 + 2) {
                    named_bar(1, 128);
                    ++passed;
                }
                S3ACC(cbar, t_cb);
            }
            if ((s & 3) == 0 && s / 4 >= Y.nres) {           // result slot of chunk s / 4 is free
                if (lane == 0) bulk_wait_read0();
                __syncwarp();
            }
            const bool act = onl && c >= 0 && c < T0;
            double xu = 0.0, xs = 0.0, xb = 0.0;             // x-edge results of lane 0's column (warp X)
            if (xe_box) {
                lds2u(xe_a + 32 * (s & 15), xu, xs);
                xb = lds1u(xe_a + 32 * (s & 15) + 16);
            }
            // ---- the neighbours' new values (previous step)
            const double S = shfl_up_w(u, 1), B = shfl_up_w(u, T1);
            const double Sq = shfl_up_w(sS, 1), Bq = shfl_up_w(sB, T1);
            // ---- rows in axis order x, y, z without the pair axis; the 2 x 2 pair (ge_solve_k<2>)
            const double rp = fma(co.e2, B, fma(co.e1, S, fma(co.c0, W, co.r0)));
            const double rq = fma(co.f2, Bq, fma(co.f1, Sq, fma(co.d0, Wq, co.q0)));
            const double ra = qf ? rq : rp, rb = qf ? rp : rq;
            fl |= act && !(pre0 && c == 0) && co.sing;
            const double ub = fma(co.mba, ra, rb) * co.inv;
            const double ua = fma(co.mab, ub, ra);
            double un = qf ? ub : ua, pv = qf ? ua : ub;
            double nS = pv, nB = pv, nWq = pv;
            {
                const bool use = xedge && s >= 1 && s < T0;
                un = use ? xu : un;
                nS = use ? xs : nS;
                nB = use ? xb : nB;
            }
            if (pre0 && c == 0) {
                un = u0;
                nS = sS0;
                nB = sB0;
                nWq = wq0;
            }
            // ---- results, state for the next step (idle lanes forward zeros: finite values only)
            sts1u_if(res_a + 8 * (((c >> 2) & (Y.nres - 1)) * Y.ressz + (sx ? 3 - (c & 3) : (c & 3))), un, act);
            W = act ? un : W;
            Wq = act ? nWq : Wq;
            u = act ? un : 0.0;
            sS = act ? nS : 0.0;
            sB = act ? nB : 0.0;
            if (c >= 0) {
                po = po + 1 == Do ? 0 : po + 1;
                pp = pp + 1 == Dp ? 0 : pp + 1;
            }
            // next step's entries (idle lanes read stale ones: never stored or forwarded)
            prep(co);
            // ---- result chunk q complete: all lanes passed its last column
            const int qd = s - lag - 3;
            if (qd >= 0 && (qd & 3) == 0 && qd / 4 < NQ) {
                const int q = qd / 4;
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    tma_store_3d(&mOUT, sx ? X0 + T0 - 2 - 4 * q : X0 + 2 + 4 * q, Y0 + 2, Z0 + 2,
                                 res + (q & (Y.nres - 1)) * Y.ressz);
                    bulk_commit();
                }
            }
        }
        while (passed < MLAST) {
            named_bar(1, 128);
            ++passed;
        }
        if (lane == 0) bulk_wait_all();
#ifdef SW_TRACE
        S3ADD(10, cbar, 0);
        S3ADD(11, sw_clock() - t_cb0, 0);
        S3ADD(12, sw_clock() - t_start, 0);
#endif
    }
    if (fl) atomicOr(A.flag, 1);
}

// ------------------------------------------------------------------------------------- host
// false if the box is not supported by the streaming engine
inline bool sweep3s_layout(const Geo &G, bool faces, bool has_aux, bool tri, Sweep3sArgs &A, size_t &smem) {
    const int T0 = G.T[0], T1 = G.T[1], T2 = G.T[2];
    if (G.dim != 3 || T0 % 4 != 0 || T0 < 4 || T1 * T2 > 32 || T1 < 1 || T2 < 1 || G.off[0] != 0 || G.off[1] != 0)
        return false;
    if (T1 + T2 > 13) return false;                          // ring depth / result ring bounds
    const Lay3 L = lay3(T1, T2, faces, has_aux);
    for (int a = 0; a < 5; ++a) {
        A.R[a] = L.R[a];
        A.Q[a] = L.Q[a];
    }
    A.has_aux = has_aux;
    smem = (size_t)L.smem;
    (void)tri;
    return smem <= 227 * 1024;
}

inline bool encode_3d(CUtensorMap *m, const double *base, int64_t pad0, int64_t pad1, int64_t pad2, int b0, int b1,
                      int b2) {
    EncodeTiledFn enc = get_encode();
    if (!enc || !base) return false;
    cuuint64_t dims[3] = {(cuuint64_t)pad0, (cuuint64_t)pad1, (cuuint64_t)pad2};
    cuuint64_t strides[2] = {(cuuint64_t)(pad0 * sizeof(double)), (cuuint64_t)(pad0 * pad1 * sizeof(double))};
    cuuint32_t box[3] = {(cuuint32_t)b0, (cuuint32_t)b1, (cuuint32_t)b2};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void *)base, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// maps[0..4] = XO, BB, F0, F1, F2 windows (box (4, R, Q)), maps[5] = the output (4, T1, T2)
template <bool FACES, bool TRI, int SHAPE>
inline cudaError_t launch_sweep3s_t(const Sweep3sArgs &A, const CUtensorMap *M, size_t smem, unsigned tiles,
                                    cudaStream_t s) {
    auto kern = k_sweep3s<FACES, TRI, SHAPE>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<tiles, 128, smem, s>>>(A, M[0], M[1], M[2], M[3], M[4], M[5]);
    return cudaGetLastError();
}

template <bool FACES, bool TRI>
inline cudaError_t launch_sweep3s_s(const Sweep3sArgs &A, const CUtensorMap *M, size_t smem, unsigned tiles,
                                    cudaStream_t s) {
    const bool c5 = A.G.T[0] == 32 && A.G.T[1] == 8 && A.G.T[2] == 4;
    return c5 ? launch_sweep3s_t<FACES, TRI, 1>(A, M, smem, tiles, s) : launch_sweep3s_t<FACES, TRI, 0>(A, M, smem, tiles, s);
}

inline cudaError_t launch_sweep3s(const Sweep3sArgs &A, const CUtensorMap *M, size_t smem, bool faces, cudaStream_t s) {
    const unsigned tiles = (unsigned)((int64_t)A.G.nt[0] * A.G.nt[1] * A.G.nt[2]);
    if (faces) return A.tri ? launch_sweep3s_s<true, true>(A, M, smem, tiles, s) : launch_sweep3s_s<true, false>(A, M, smem, tiles, s);
    return A.tri ? launch_sweep3s_s<false, true>(A, M, smem, tiles, s) : launch_sweep3s_s<false, false>(A, M, smem, tiles, s);
}

}  // namespace sw
