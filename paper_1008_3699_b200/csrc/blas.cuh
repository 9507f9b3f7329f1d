// blas.cuh -- PCG vector kernels with fused, deterministic reductions (north_star
// "PCG driver with fused dot-product/axpy reductions").
//
// Every reduction writes one partial per CTA (fixed thread order inside the CTA) and a
// single-CTA finisher sums the partials in CTA order, so results are bitwise
// reproducible run to run.  Interior nodes are addressed by a flattened local index;
// ghost layers of the padded arrays are never written here.
#pragma once
#include "common.cuh"

namespace sw {

constexpr int RED_THREADS = 256;
// Grid size of the row-segment / reduction kernels: 8 CTAs per SM of the current device (1184 on
// a 148-SM B200), queried once per process, so every reduction of a run has one fixed order.
inline int red_blocks() {
    static const int v = [] {
        int dev = 0, sms = 0;
        if (cudaGetDevice(&dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms < 1)
            sms = 148;
        return 8 * sms;
    }();
    return v;
}

// Accurate reductions: every dot product is accumulated in double-double (TwoProd by fma,
// TwoSum), per thread, then per CTA in fixed warp-shuffle order, then across CTAs in CTA
// order; the final hi + lo is the correctly rounded exact sum except in near-tie cases,
// which makes PCG iterates independent of the reduction tree (PCG parity).
struct DD {
    double hi, lo;
};

__device__ inline void dd_add(DD &s, double p) {
    double t = s.hi + p;
    double bp = t - s.hi;
    double err = (s.hi - (t - bp)) + (p - bp);
    s.hi = t;
    s.lo += err;
}

__device__ inline void dd_add_prod(DD &s, double a, double b) {
    double p = a * b;
    double e = fma(a, b, -p);
    dd_add(s, p);
    s.lo += e;
}

__device__ inline DD dd_merge(DD a, DD b) {
    DD r = a;
    dd_add(r, b.hi);
    r.lo += b.lo;
    double t = r.hi + r.lo;          // renormalise
    r.lo = r.lo - (t - r.hi);
    r.hi = t;
    return r;
}

__device__ inline DD block_sum_dd(DD v, DD *sh) {
    for (int o = 16; o > 0; o >>= 1) {
        DD w;
        w.hi = __shfl_down_sync(0xffffffffu, v.hi, o);
        w.lo = __shfl_down_sync(0xffffffffu, v.lo, o);
        v = dd_merge(v, w);
    }
    int wi = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) sh[wi] = v;
    __syncthreads();
    DD s = {0.0, 0.0};
    if (threadIdx.x == 0)
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s = dd_merge(s, sh[i]);
    __syncthreads();
    return s;
}

__device__ inline int64_t interior_index(const Geo &G, int64_t t) {
    int64_t i0 = t % G.n[0];
    int64_t r = t / G.n[0];
    int64_t i1 = r % G.n[1];
    int64_t i2 = r / G.n[1];
    return G.origin + i0 + G.P0 * i1 + G.P01 * i2;
}

// (A x)_p = a_P x_p - sum_q c_pq x_q, evaluated s = a_P x_p; s = fma(-c, x_q, s) in axis
// order (-, +) (DESIGN R-7, same as the oracle).  Ghost neighbours read 0.
__device__ inline double apply_A_at(const Geo &G, const double *const F[3], const double *x, int64_t idx,
                                    const int64_t g[3]) {
    double s = a_p(G, F, g) * x[idx];
    const int64_t st[3] = {1, G.P0, G.P01};
    for (int a = 0; a < G.dim; ++a) {
        s = fma(-face(G, F, g, a, -1), x[idx - st[a]], s);
        s = fma(-face(G, F, g, a, +1), x[idx + st[a]], s);
    }
    return s;
}

__device__ inline void local_to_global(const Geo &G, int64_t t, int64_t g[3]) {
    g[0] = t % G.n[0];
    int64_t r = t / G.n[0];
    g[1] = r % G.n[1];
    g[2] = r / G.n[1];
    for (int a = 0; a < 3; ++a) g[a] += G.off[a];
}

// q = A p ; partial[blk] = sum p.q
__global__ void k_spmv_dot(Geo G, const double *F0, const double *F1, const double *F2, const double *p, double *q,
                           DD *partial) {
    __shared__ DD sh[RED_THREADS / 32];
    const double *F[3] = {F0, F1, F2};
    int64_t N = G.n[0] * G.n[1] * G.n[2];
    DD acc = {0.0, 0.0};
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < N; t += (int64_t)gridDim.x * blockDim.x) {
        int64_t g[3];
        local_to_global(G, t, g);
        int64_t i = interior_index(G, t);
        double v = apply_A_at(G, F, p, i, g);
        q[i] = v;
        dd_add_prod(acc, p[i], v);
    }
    DD s = block_sum_dd(acc, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

// r = b - A x ; partial[2*blk] = sum r.r, partial[2*blk+1] = sum b.b
__global__ void k_residual(Geo G, const double *F0, const double *F1, const double *F2, const double *x,
                           const double *b, double *r, DD *partial) {
    __shared__ DD sh[RED_THREADS / 32];
    const double *F[3] = {F0, F1, F2};
    int64_t N = G.n[0] * G.n[1] * G.n[2];
    DD rr = {0.0, 0.0}, bb = {0.0, 0.0};
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < N; t += (int64_t)gridDim.x * blockDim.x) {
        int64_t g[3];
        local_to_global(G, t, g);
        int64_t i = interior_index(G, t);
        double v = b[i] - apply_A_at(G, F, x, i, g);
        if (r) r[i] = v;
        dd_add_prod(rr, v, v);
        dd_add_prod(bb, b[i], b[i]);
    }
    DD s1 = block_sum_dd(rr, sh);
    DD s2 = block_sum_dd(bb, sh);
    if (threadIdx.x == 0) {
        partial[2 * blockIdx.x] = s1;
        partial[2 * blockIdx.x + 1] = s2;
    }
}

// generic dot: partial[blk] = sum a.b
__global__ void k_dot(Geo G, const double *a, const double *b, DD *partial) {
    __shared__ DD sh[RED_THREADS / 32];
    int64_t N = G.n[0] * G.n[1] * G.n[2];
    DD acc = {0.0, 0.0};
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < N; t += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = interior_index(G, t);
        dd_add_prod(acc, a[i], b[i]);
    }
    DD s = block_sum_dd(acc, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

// ---------------------------------------------------------------------------------------
// Row-segment kernels (the PCG hot path): a work item is a segment of up to 2*RSEG interior
// nodes of one grid row (x fastest); thread i of the CTA handles nodes i and i + RSEG of the
// segment, so every access is a fully coalesced row run and no thread divides by the row
// length.  CTAs stride over items in a fixed order and write one double-double partial each,
// so every reduction is deterministic for a given launch shape.
constexpr int RSEG = RED_THREADS;               // double2 per item and CTA

struct Rows {
    int64_t n0, n1, rows, segs, items;          // interior row length, rows, segments per row
    int64_t P0, P01, origin;
};

__host__ __device__ inline Rows make_rows(const Geo &G) {
    Rows R;
    R.n0 = G.n[0];
    R.n1 = G.n[1];
    R.rows = G.n[1] * G.n[2];
    R.segs = (G.n[0] + 2 * RSEG - 1) / (2 * RSEG);
    R.items = R.rows * R.segs;
    R.P0 = G.P0;
    R.P01 = G.P01;
    R.origin = G.origin;
    return R;
}

// padded index of (x, row)
__device__ inline int64_t row_base(const Rows &R, int64_t row) {
    const int64_t y = row % R.n1, z = row / R.n1;
    return R.origin + y * R.P0 + z * R.P01;
}

// (A x)_p as in the oracle: s = a_P x_p, then s = fma(-c, x_q, s) over x-, x+, y-, y+, z-, z+
template <int DIM, bool FACES>
__device__ __forceinline__ double apply_A_fast(const double *__restrict__ F0, const double *__restrict__ F1,
                                               const double *__restrict__ F2, const double *__restrict__ x,
                                               int64_t i, int64_t P0, int64_t P01, double beta) {
    double c0 = 1.0, c1 = 1.0, c2 = 1.0, c3 = 1.0, c4 = 1.0, c5 = 1.0;
    if (FACES) {
        c0 = F0[i]; c1 = F0[i + 1];
        if (DIM > 1) { c2 = F1[i]; c3 = F1[i + P0]; }
        if (DIM > 2) { c4 = F2[i]; c5 = F2[i + P01]; }
    }
    double ap = c0 + c1;
    if (DIM > 1) ap = ap + (c2 + c3);
    if (DIM > 2) ap = ap + (c4 + c5);
    ap = ap + beta;
    double s = ap * x[i];
    s = fma(-c0, x[i - 1], s);
    s = fma(-c1, x[i + 1], s);
    if (DIM > 1) {
        s = fma(-c2, x[i - P0], s);
        s = fma(-c3, x[i + P0], s);
    }
    if (DIM > 2) {
        s = fma(-c4, x[i - P01], s);
        s = fma(-c5, x[i + P01], s);
    }
    return s;
}

// q = A p ; partial[blk] = sum p.q
template <int DIM, bool FACES>
__global__ void __launch_bounds__(RED_THREADS) k_spmv_dot_r(Rows R, double beta, const double *__restrict__ F0,
                                                            const double *__restrict__ F1,
                                                            const double *__restrict__ F2,
                                                            const double *__restrict__ p, double *__restrict__ q,
                                                            DD *partial) {
    __shared__ DD sh[RED_THREADS / 32];
    DD acc = {0.0, 0.0};
    for (int64_t it = blockIdx.x; it < R.items; it += gridDim.x) {
        const int64_t row = it / R.segs, seg = it % R.segs;
        const int64_t xb = seg * 2 * RSEG + threadIdx.x;
        const int64_t b = row_base(R, row);
        for (int h = 0; h < 2; ++h) {
            const int64_t x = xb + h * RSEG;
            if (x < R.n0) {
                const int64_t i = b + x;
                const double v = apply_A_fast<DIM, FACES>(F0, F1, F2, p, i, R.P0, R.P01, beta);
                q[i] = v;
                dd_add_prod(acc, p[i], v);
            }
        }
    }
    DD sm = block_sum_dd(acc, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = sm;
}

// The PCG direction update fused into the next SpMV: p_new = z + beta p_old at
// the node and its stencil neighbours (each value exactly as k_pupdate_r computes it), q = A p_new,
// p_new stored (a second buffer: other threads still read p_old), partial[blk] = sum p_new.q.
template <int DIM, bool FACES>
__global__ void __launch_bounds__(RED_THREADS) k_pspmv_dot_r(Rows R, double beta_a, const double *beta_dev,
                                                             const double *__restrict__ F0,
                                                             const double *__restrict__ F1,
                                                             const double *__restrict__ F2,
                                                             const double *__restrict__ z,
                                                             const double *pold_a, double *pnew_a,
                                                             double *__restrict__ q, DD *partial,
                                                             const int *par_dev = nullptr) {
    __shared__ DD sh[RED_THREADS / 32];
    const double be = *beta_dev;
    // par_dev (a device-resident PCG loop): odd parity swaps the two direction buffers
    const bool sw_ = par_dev && *par_dev;
    const double *const pold = sw_ ? pnew_a : pold_a;
    double *const pnew = sw_ ? const_cast<double *>(pold_a) : pnew_a;
    auto P = [&](int64_t j) { return fma(be, pold[j], z[j]); };
    DD acc = {0.0, 0.0};
    for (int64_t it = blockIdx.x; it < R.items; it += gridDim.x) {
        const int64_t row = it / R.segs, seg = it % R.segs;
        const int64_t xb = seg * 2 * RSEG + threadIdx.x;
        const int64_t b = row_base(R, row);
        for (int h = 0; h < 2; ++h) {
            const int64_t x = xb + h * RSEG;
            if (x < R.n0) {
                const int64_t i = b + x;
                double c0 = 1.0, c1 = 1.0, c2 = 1.0, c3 = 1.0, c4 = 1.0, c5 = 1.0;
                if (FACES) {
                    c0 = F0[i]; c1 = F0[i + 1];
                    if (DIM > 1) { c2 = F1[i]; c3 = F1[i + R.P0]; }
                    if (DIM > 2) { c4 = F2[i]; c5 = F2[i + R.P01]; }
                }
                double ap = c0 + c1;
                if (DIM > 1) ap = ap + (c2 + c3);
                if (DIM > 2) ap = ap + (c4 + c5);
                ap = ap + beta_a;
                const double pi = P(i);
                double v = ap * pi;
                v = fma(-c0, P(i - 1), v);
                v = fma(-c1, P(i + 1), v);
                if (DIM > 1) {
                    v = fma(-c2, P(i - R.P0), v);
                    v = fma(-c3, P(i + R.P0), v);
                }
                if (DIM > 2) {
                    v = fma(-c4, P(i - R.P01), v);
                    v = fma(-c5, P(i + R.P01), v);
                }
                pnew[i] = pi;
                q[i] = v;
                dd_add_prod(acc, pi, v);
            }
        }
    }
    DD sm = block_sum_dd(acc, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = sm;
}

// 3D form of k_pspmv_dot_r that marches z: a block owns 32 x 8 columns, keeps p_new of the planes
// z-1, z, z+1 in registers and the x / y neighbours of plane z in shared memory, so every value of
// p_old, z and the faces is read from DRAM once and p_new = z + beta p_old is formed once per node
// (the row kernel re-reads the planes z +- 1, 1.5x the algorithmic bytes).  q and p_new are the
// same operations in the same order as k_pspmv_dot_r (bitwise equal); the per-block partial sums
// follow the block's own (fixed) order.
#ifndef SW_ZC
#define SW_ZC 8
#endif
template <bool FACES>
__global__ void __launch_bounds__(256) k_pspmv3_zm(Rows R, double beta_a, const double *beta_dev,
                                                   const double *__restrict__ F0, const double *__restrict__ F1,
                                                   const double *__restrict__ F2, const double *__restrict__ z,
                                                   const double *pold_a, double *pnew_a,
                                                   double *__restrict__ q, DD *partial, const int *par_dev = nullptr) {
    constexpr int TX = 32, TY = 8;
    __shared__ double tile[2][TY + 2][TX + 2];
    __shared__ DD sh[256 / 32];
    const double be = *beta_dev;
    const bool sw_ = par_dev && *par_dev;
    const double *const pold = sw_ ? pnew_a : pold_a;
    double *const pnew = sw_ ? const_cast<double *>(pold_a) : pnew_a;
    auto P = [&](int64_t j) { return fma(be, pold[j], z[j]); };
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    constexpr int ZC = SW_ZC;                 // planes per work item (more items in flight)
    const int64_t ntx = (R.n0 + TX - 1) / TX, nty = (R.n1 + TY - 1) / TY, n2 = R.rows / R.n1;
    const int64_t nzc = (n2 + ZC - 1) / ZC;
    DD acc = {0.0, 0.0};
    for (int64_t t = blockIdx.x; t < ntx * nty * nzc; t += gridDim.x) {
        const int64_t tc = t % (ntx * nty), z0 = (t / (ntx * nty)) * ZC;
        const int64_t z1 = z0 + ZC < n2 ? z0 + ZC : n2;
        const int64_t x = (tc % ntx) * TX + tx, y = (tc / ntx) * TY + ty;
        const bool in = x < R.n0 && y < R.n1;
        const bool hx = in && (tx == TX - 1 || x == R.n0 - 1), hy = in && (ty == TY - 1 || y == R.n1 - 1);
        int64_t i = R.origin + (in ? y : 0) * R.P0 + (in ? x : 0) + z0 * R.P01;
        double Pm = P(i - R.P01), Pc = P(i);
        double f4 = FACES ? F2[i] : 1.0;
        for (int64_t k = z0; k < z1; ++k) {
            const int b = (int)(k & 1);
            const double Pp = P(i + R.P01);
            double c0 = 1.0, c1 = 1.0, c2 = 1.0, c3 = 1.0, c5 = 1.0;
            if (FACES) { c0 = F0[i]; c1 = F0[i + 1]; c2 = F1[i]; c3 = F1[i + R.P0]; c5 = F2[i + R.P01]; }
            if (in) {
                tile[b][ty + 1][tx + 1] = Pc;
                if (tx == 0) tile[b][ty + 1][0] = P(i - 1);
                if (hx) tile[b][ty + 1][tx + 2] = P(i + 1);
                if (ty == 0) tile[b][0][tx + 1] = P(i - R.P0);
                if (hy) tile[b][ty + 2][tx + 1] = P(i + R.P0);
            }
            __syncthreads();
            if (in) {
                const double c4 = f4;
                double ap = c0 + c1;
                ap = ap + (c2 + c3);
                ap = ap + (c4 + c5);
                ap = ap + beta_a;
                double v = ap * Pc;
                v = fma(-c0, tile[b][ty + 1][tx], v);
                v = fma(-c1, tile[b][ty + 1][tx + 2], v);
                v = fma(-c2, tile[b][ty][tx + 1], v);
                v = fma(-c3, tile[b][ty + 2][tx + 1], v);
                v = fma(-c4, Pm, v);
                v = fma(-c5, Pp, v);
                pnew[i] = Pc;
                q[i] = v;
                dd_add_prod(acc, Pc, v);
            }
            Pm = Pc;
            Pc = Pp;
            f4 = c5;
            i += R.P01;
        }
        __syncthreads();                      // the next tile reuses the buffers
    }
    DD sm = block_sum_dd(acc, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = sm;
}

// out = r - A x (interior nodes): the residual of a multigrid level in one pass (the same values as
// k_spmv_dot_r followed by k_sub_r with theta = 1)
template <int DIM, bool FACES>
__global__ void __launch_bounds__(RED_THREADS) k_resid_r(Rows R, double beta, const double *__restrict__ F0,
                                                         const double *__restrict__ F1, const double *__restrict__ F2,
                                                         const double *__restrict__ x, const double *__restrict__ r,
                                                         double *__restrict__ out) {
    for (int64_t it = blockIdx.x; it < R.items; it += gridDim.x) {
        const int64_t row = it / R.segs, seg = it % R.segs;
        const int64_t xb = seg * 2 * RSEG + threadIdx.x;
        const int64_t b = row_base(R, row);
        for (int h = 0; h < 2; ++h) {
            const int64_t xx = xb + h * RSEG;
            if (xx < R.n0) {
                const int64_t i = b + xx;
                out[i] = __dsub_rn(r[i], apply_A_fast<DIM, FACES>(F0, F1, F2, x, i, R.P0, R.P01, beta));
            }
        }
    }
}

// partial[blk] = sum a.b
__global__ void __launch_bounds__(RED_THREADS) k_dot_r(Rows R, const double *__restrict__ a,
                                                       const double *__restrict__ b, DD *partial) {
    __shared__ DD sh[RED_THREADS / 32];
    DD acc = {0.0, 0.0};
    for (int64_t it = blockIdx.x; it < R.items; it += gridDim.x) {
        const int64_t row = it / R.segs, seg = it % R.segs;
        const int64_t xb = seg * 2 * RSEG + threadIdx.x;
        const int64_t base = row_base(R, row);
        for (int h = 0; h < 2; ++h)
            if (xb + h * RSEG < R.n0) dd_add_prod(acc, a[base + xb + h * RSEG], b[base + xb + h * RSEG]);
    }
    DD sm = block_sum_dd(acc, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = sm;
}

// partial = sum z.(r - rold), the difference rounded first (the oracle's rold = r - rold, then z.rold)
__global__ void __launch_bounds__(RED_THREADS) k_dot_diff_r(Rows R, const double *__restrict__ z,
                                                            const double *__restrict__ r,
                                                            const double *__restrict__ rold, DD *partial) {
    __shared__ DD sh[RED_THREADS / 32];
    DD acc = {0.0, 0.0};
    for (int64_t it = blockIdx.x; it < R.items; it += gridDim.x) {
        const int64_t row = it / R.segs, seg = it % R.segs;
        const int64_t xb = seg * 2 * RSEG + threadIdx.x;
        const int64_t base = row_base(R, row);
        for (int h = 0; h < 2; ++h) {
            const int64_t i = base + xb + h * RSEG;
            if (xb + h * RSEG < R.n0) dd_add_prod(acc, z[i], __dsub_rn(r[i], rold[i]));
        }
    }
    DD sm = block_sum_dd(acc, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = sm;
}

// x = fma(alpha, p, x) ; r = fma(-alpha, q, r) ; partial = sum r.r
__global__ void __launch_bounds__(RED_THREADS) k_axpy2_dot_r(Rows R, const double *alpha_dev, double *__restrict__ x,
                                                             double *__restrict__ r, const double *p_a,
                                                             const double *__restrict__ q, DD *partial,
                                                             const double *p_b = nullptr, const int *par_dev = nullptr) {
    __shared__ DD sh[RED_THREADS / 32];
    const double al = *alpha_dev;
    const double *const p = (par_dev && *par_dev) ? p_b : p_a;   // (device-resident PCG: the current direction)
    DD acc = {0.0, 0.0};
    for (int64_t it = blockIdx.x; it < R.items; it += gridDim.x) {
        const int64_t row = it / R.segs, seg = it % R.segs;
        const int64_t xb = seg * 2 * RSEG + threadIdx.x;
        const int64_t base = row_base(R, row);
        for (int h = 0; h < 2; ++h) {
            if (xb + h * RSEG < R.n0) {
                const int64_t i = base + xb + h * RSEG;
                x[i] = fma(al, p[i], x[i]);
                const double rv = fma(-al, q[i], r[i]);
                r[i] = rv;
                dd_add_prod(acc, rv, rv);
            }
        }
    }
    DD sm = block_sum_dd(acc, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = sm;
}

// p = fma(beta, p, z)   (first: p = z)
__global__ void __launch_bounds__(RED_THREADS) k_pupdate_r(Rows R, const double *beta_dev, int first,
                                                           const double *__restrict__ z, double *__restrict__ p) {
    const double be = first ? 0.0 : *beta_dev;
    for (int64_t it = blockIdx.x; it < R.items; it += gridDim.x) {
        const int64_t row = it / R.segs, seg = it % R.segs;
        const int64_t xb = seg * 2 * RSEG + threadIdx.x;
        const int64_t base = row_base(R, row);
        for (int h = 0; h < 2; ++h) {
            if (xb + h * RSEG < R.n0) {
                const int64_t i = base + xb + h * RSEG;
                p[i] = first ? z[i] : fma(be, p[i], z[i]);
            }
        }
    }
}

// y = r - theta q (interior nodes; the m-step preconditioner's residual), product and difference
// rounded separately (no contraction)
__global__ void __launch_bounds__(RED_THREADS) k_sub_r(Rows R, const double *__restrict__ r, double theta,
                                                       const double *__restrict__ q, double *__restrict__ y) {
    for (int64_t it = blockIdx.x; it < R.items; it += gridDim.x) {
        const int64_t row = it / R.segs, seg = it % R.segs;
        const int64_t xb = seg * 2 * RSEG + threadIdx.x;
        const int64_t base = row_base(R, row);
        for (int h = 0; h < 2; ++h)
            if (xb + h * RSEG < R.n0) {
                const int64_t i = base + xb + h * RSEG;
                y[i] = __dsub_rn(r[i], __dmul_rn(theta, q[i]));
            }
    }
}

// z += d (interior nodes)
__global__ void __launch_bounds__(RED_THREADS) k_addto_r(Rows R, double *__restrict__ z, const double *__restrict__ d) {
    for (int64_t it = blockIdx.x; it < R.items; it += gridDim.x) {
        const int64_t row = it / R.segs, seg = it % R.segs;
        const int64_t xb = seg * 2 * RSEG + threadIdx.x;
        const int64_t base = row_base(R, row);
        for (int h = 0; h < 2; ++h)
            if (xb + h * RSEG < R.n0) {
                const int64_t i = base + xb + h * RSEG;
                z[i] = z[i] + d[i];
            }
    }
}

// x = s x (interior nodes)
__global__ void __launch_bounds__(RED_THREADS) k_scale_r(Rows R, double sc, double *__restrict__ x) {
    for (int64_t it = blockIdx.x; it < R.items; it += gridDim.x) {
        const int64_t row = it / R.segs, seg = it % R.segs;
        const int64_t xb = seg * 2 * RSEG + threadIdx.x;
        const int64_t base = row_base(R, row);
        for (int h = 0; h < 2; ++h)
            if (xb + h * RSEG < R.n0) {
                const int64_t i = base + xb + h * RSEG;
                x[i] = sc * x[i];
            }
    }
}

// out = a x + b y (interior nodes), products and sum rounded separately; out may alias x or y
__global__ void __launch_bounds__(RED_THREADS) k_axpby_r(Rows R, double a, const double *x, double b, const double *y,
                                                         double *out) {
    for (int64_t it = blockIdx.x; it < R.items; it += gridDim.x) {
        const int64_t row = it / R.segs, seg = it % R.segs;
        const int64_t xb = seg * 2 * RSEG + threadIdx.x;
        const int64_t base = row_base(R, row);
        for (int h = 0; h < 2; ++h)
            if (xb + h * RSEG < R.n0) {
                const int64_t i = base + xb + h * RSEG;
                out[i] = __dadd_rn(__dmul_rn(a, x[i]), __dmul_rn(b, y[i]));
            }
    }
}

// PCG scalars kept on the device
struct CgScalars {
    double rz, pq, alpha, beta, rr, bb, rz_new, zd;   // zd = z.(r_new - r_old) (flexible CG)
    int it, par, stop, pad;                           // device-resident loop: iteration, buffer parity, stop code
};

// End of one iteration of the device-resident PCG loop (a conditional WHILE node): count it, flip the
// direction-buffer parity, and keep looping while ||r|| / ||b|| >= rtol, r.r is a number and it < maxit
// (stop: 1 converged, 2 NaN, 3 maxit) -- the host loop's decisions, taken on the device.
__global__ void k_pcg_step(CgScalars *c, cudaGraphConditionalHandle h, double rtol, double bnorm, int maxit) {
    c->it += 1;
    c->par ^= 1;
    const double rel = sqrt(c->rr) / bnorm;
    int stop = 0;
    if (rel < rtol) stop = 1;
    else if (!(c->rr == c->rr)) stop = 2;
    else if (c->it >= maxit) stop = 3;
    c->stop = stop;
    cudaGraphSetConditional(h, stop == 0 ? 1u : 0u);
}

// sum `nparts` partials (stride `stride`, offset `off`) in fixed order into *dst = hi + lo
__global__ void k_finish_sum(const DD *partial, int nparts, int stride, int off, double *dst) {
    __shared__ DD sh[RED_THREADS / 32];
    DD acc = {0.0, 0.0};
    for (int i = threadIdx.x; i < nparts; i += blockDim.x) acc = dd_merge(acc, partial[(int64_t)i * stride + off]);
    DD s = block_sum_dd(acc, sh);
    if (threadIdx.x == 0) *dst = s.hi + s.lo;
}

// sum `nparts` partials in fixed order into dst[0] = hi, dst[1] = lo (double-double)
__global__ void k_finish_dd(const DD *partial, int nparts, double *dst) {
    __shared__ DD sh[RED_THREADS / 32];
    DD acc = {0.0, 0.0};
    for (int i = threadIdx.x; i < nparts; i += blockDim.x) acc = dd_merge(acc, partial[i]);
    DD s = block_sum_dd(acc, sh);
    if (threadIdx.x == 0) {
        dst[0] = s.hi;
        dst[1] = s.lo;
    }
}

// same with a stride / offset over the partials (k_residual's interleaved r.r and b.b)
__global__ void k_finish_dd_strided(const DD *partial, int nparts, int stride, int off, double *dst) {
    __shared__ DD sh[RED_THREADS / 32];
    DD acc = {0.0, 0.0};
    for (int i = threadIdx.x; i < nparts; i += blockDim.x) acc = dd_merge(acc, partial[(int64_t)i * stride + off]);
    DD s = block_sum_dd(acc, sh);
    if (threadIdx.x == 0) {
        dst[0] = s.hi;
        dst[1] = s.lo;
    }
}

__global__ void k_set_scalar(double *dst, double v) { *dst = v; }

// alpha = rz / pq
__global__ void k_cg_alpha(CgScalars *c) { c->alpha = c->rz / c->pq; }
// beta = rz_new / rz ; rz = rz_new
__global__ void k_cg_beta(CgScalars *c) {
    c->beta = c->rz_new / c->rz;
    c->rz = c->rz_new;
}

// flexible (Polak-Ribiere) beta = z+.(r+ - r) / (r.z)
__global__ void k_cg_beta_flex(CgScalars *c) {
    c->beta = c->zd / c->rz;
    c->rz = c->rz_new;
}

// x = fma(alpha, p, x) ; r = fma(-alpha, q, r) ; partial = sum r.r
__global__ void k_axpy2_dot(Geo G, const CgScalars *c, double *x, double *r, const double *p, const double *q,
                            DD *partial) {
    __shared__ DD sh[RED_THREADS / 32];
    int64_t N = G.n[0] * G.n[1] * G.n[2];
    double al = c->alpha;
    DD acc = {0.0, 0.0};
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < N; t += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = interior_index(G, t);
        x[i] = fma(al, p[i], x[i]);
        double rv = fma(-al, q[i], r[i]);
        r[i] = rv;
        dd_add_prod(acc, rv, rv);
    }
    DD s = block_sum_dd(acc, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

// p = fma(beta, p, z)   (first: p = z)
__global__ void k_pupdate(Geo G, const CgScalars *c, int first, const double *z, double *p) {
    int64_t N = G.n[0] * G.n[1] * G.n[2];
    double be = first ? 0.0 : c->beta;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < N; t += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = interior_index(G, t);
        p[i] = first ? z[i] : fma(be, p[i], z[i]);
    }
}

// faces from node diffusivities (DESIGN R-12):
//   F[a] at node g = scale_a * ((2 k(g-e_a)) k(g)) / (k(g-e_a) + k(g))
// k layout: per used axis kd[a] nodes, local coordinate c stored at c + kor[a]
// (kor = 1 with a one-node ring, 2 on the slab axis with two extra layers).
struct KLayout {
    int64_t kd[3];
    int64_t kor[3];
    double scale[3];
};

__global__ void k_faces_from_k(Geo G, KLayout K, const double *kk, double *F0, double *F1, double *F2) {
    int64_t w[3] = {1, 1, 1};
    for (int a = 0; a < G.dim; ++a) w[a] = G.n[a] + 4;
    int64_t N = w[0] * w[1] * w[2];
    double *F[3] = {F0, F1, F2};
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < N; t += (int64_t)gridDim.x * blockDim.x) {
        int64_t l[3] = {t % w[0], (t / w[0]) % w[1], t / (w[0] * w[1])};
        for (int a = 0; a < G.dim; ++a) l[a] -= 2;           // local coordinates in [-2, n+2)
        int64_t g[3] = {l[0] + G.off[0], l[1] + G.off[1], l[2] + G.off[2]};
        int64_t pi = gidx(G, g[0], g[1], g[2]);
        for (int a = 0; a < G.dim; ++a) {
            bool ok = (g[a] >= 0 && g[a] <= G.ng[a]);       // faces 0..ng along a
            for (int b = 0; b < G.dim; ++b)
                if (b != a && (g[b] < -1 || g[b] > G.ng[b])) ok = false;
            int64_t cq[3], cp[3];
            for (int b = 0; b < 3; ++b) {
                cq[b] = (b < G.dim) ? l[b] + K.kor[b] : 0;
                cp[b] = cq[b] - (b == a ? 1 : 0);
                if (b < G.dim && (cq[b] < 0 || cp[b] < 0 || cq[b] >= K.kd[b] || cp[b] >= K.kd[b])) ok = false;
            }
            double v = 0.0;
            if (ok) {
                double kp = kk[cp[0] + K.kd[0] * (cp[1] + K.kd[1] * cp[2])];
                double kq = kk[cq[0] + K.kd[0] * (cq[1] + K.kd[1] * cq[2])];
                v = K.scale[a] * ((2.0 * kp) * kq / (kp + kq));
            }
            F[a][pi] = v;
        }
    }
}

}  // namespace sw
