// mg.cuh -- grid transfer kernels of the geometric multigrid preconditioner:
// piecewise-constant aggregation of the 2^k fine nodes that share a coarse node (k = number of
// coarsened axes; all axes, or the strongly coupled ones only for anisotropic problems), R = P^T,
// and the Galerkin coarse operator R A P, which is again a face-coefficient operator: each coarse
// face is the sum of the fine faces it covers, beta_c = 2^k beta (DESIGN R-19).  Every sum is
// pairwise along the coarsened axes in ascending order (pairs along the first, then pairs of
// pairs along the next), mirrored by the oracle-side composition in tests/test_gpu_mg.py.
#pragma once
#include "common.cuh"
#include "blas.cuh"

namespace sw {

// the coarsened axes of one level (bit a of `mask`), their fine strides and the node ratio per axis
struct Coarsen {
    int mask;
    int k;             // number of coarsened axes
    int ax[3];         // the coarsened axes, ascending
};

__host__ __device__ inline Coarsen make_coarsen(int mask, int dim) {
    Coarsen c{};
    c.mask = mask;
    for (int a = 0; a < dim; ++a)
        if ((mask >> a) & 1) c.ax[c.k++] = a;
    return c;
}

// pairwise sum of v(offset) over the 2^k offsets spanned by strides s[0..k-1] (s[0] fastest)
template <typename V>
__device__ __forceinline__ double agg_sum(int k, const int64_t s[3], V v) {
    if (k == 0) return v(0);
    if (k == 1) return v(0) + v(s[0]);
    const double lo = (v(0) + v(s[0])) + (v(s[1]) + v(s[1] + s[0]));
    if (k == 2) return lo;
    return lo + ((v(s[2]) + v(s[2] + s[0])) + (v(s[2] + s[1]) + v(s[2] + s[1] + s[0])));
}

__device__ __forceinline__ int64_t axis_stride(const Geo &G, int a) { return a == 0 ? 1 : (a == 1 ? G.P0 : G.P01); }

// coarse face along axis a at coarse node I (I_a in [0, nc_a], the other axes in [0, nc_b)): the
// sum of the fine faces at fine position r_a I_a along a over the coarsened axes other than a
__global__ void k_coarsen_faces(Geo Gf, Geo Gc, Coarsen C, int a, const double *__restrict__ Ff,
                                double *__restrict__ Fc) {
    int64_t m[3] = {1, 1, 1};
    for (int b = 0; b < Gc.dim; ++b) m[b] = Gc.n[b] + (b == a ? 1 : 0);
    const int64_t total = m[0] * m[1] * m[2];
    int k = 0;
    int64_t s[3] = {0, 0, 0};
    for (int t = 0; t < C.k; ++t)
        if (C.ax[t] != a) s[k++] = axis_stride(Gf, C.ax[t]);
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t I[3] = {e % m[0], (e / m[0]) % m[1], e / (m[0] * m[1])};
        int64_t f[3];
        for (int b = 0; b < 3; ++b) f[b] = ((C.mask >> b) & 1) ? 2 * I[b] : I[b];
        const int64_t i0 = gidx(Gf, f[0] + Gf.off[0], f[1] + Gf.off[1], f[2] + Gf.off[2]);
        const double v = agg_sum(k, s, [&](int64_t d) { return Ff ? Ff[i0 + d] : 1.0; });
        Fc[gidx(Gc, I[0] + Gc.off[0], I[1] + Gc.off[1], I[2] + Gc.off[2])] = v;
    }
}

// first fine node of coarse node I
__device__ __forceinline__ int64_t fine_first(const Geo &Gf, const Coarsen &C, const int64_t I[3]) {
    int64_t f[3];
    for (int b = 0; b < 3; ++b) f[b] = ((C.mask >> b) & 1) ? 2 * I[b] : I[b];
    return gidx(Gf, f[0] + Gf.off[0], f[1] + Gf.off[1], f[2] + Gf.off[2]);
}

// r_c[I] = sum of r over the fine nodes of I
__global__ void k_restrict(Geo Gf, Geo Gc, Coarsen C, const double *__restrict__ rf, double *__restrict__ rc) {
    const int64_t total = Gc.n[0] * Gc.n[1] * Gc.n[2];
    int64_t s[3] = {0, 0, 0};
    for (int t = 0; t < C.k; ++t) s[t] = axis_stride(Gf, C.ax[t]);
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t I[3] = {e % Gc.n[0], (e / Gc.n[0]) % Gc.n[1], e / (Gc.n[0] * Gc.n[1])};
        const int64_t i = fine_first(Gf, C, I);
        rc[gidx(Gc, I[0] + Gc.off[0], I[1] + Gc.off[1], I[2] + Gc.off[2])] =
            agg_sum(C.k, s, [&](int64_t d) { return rf[i + d]; });
    }
}

// r_c[I] = sum over the fine nodes of I of (r - A x), in k_restrict's order: the residual of the
// pre-smoothed iterate restricted in one pass (each fine residual as k_resid_r computes it)
template <int DIM, bool FACES>
__global__ void k_resid_restrict(Geo Gf, Geo Gc, Coarsen C, double beta, const double *__restrict__ F0,
                                 const double *__restrict__ F1, const double *__restrict__ F2,
                                 const double *__restrict__ x, const double *__restrict__ r, double *__restrict__ rc) {
    const int64_t total = Gc.n[0] * Gc.n[1] * Gc.n[2];
    int64_t s[3] = {0, 0, 0};
    for (int t = 0; t < C.k; ++t) s[t] = axis_stride(Gf, C.ax[t]);
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t I[3] = {e % Gc.n[0], (e / Gc.n[0]) % Gc.n[1], e / (Gc.n[0] * Gc.n[1])};
        const int64_t i = fine_first(Gf, C, I);
        rc[gidx(Gc, I[0] + Gc.off[0], I[1] + Gc.off[1], I[2] + Gc.off[2])] = agg_sum(C.k, s, [&](int64_t d) {
            return __dsub_rn(r[i + d], apply_A_fast<DIM, FACES>(F0, F1, F2, x, i + d, Gf.P0, Gf.P01, beta));
        });
    }
}

// x[i] += s x_c[parent(i)]  (product and sum rounded separately; s = 1 adds x_c)
__global__ void k_prolong_add(Geo Gf, Geo Gc, Coarsen C, double sc, const double *__restrict__ xc,
                              double *__restrict__ xf) {
    const int64_t total = Gf.n[0] * Gf.n[1] * Gf.n[2];
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i[3] = {e % Gf.n[0], (e / Gf.n[0]) % Gf.n[1], e / (Gf.n[0] * Gf.n[1])};
        int64_t I[3];
        for (int b = 0; b < 3; ++b) I[b] = ((C.mask >> b) & 1) ? i[b] / 2 : i[b];
        const int64_t fi = gidx(Gf, i[0] + Gf.off[0], i[1] + Gf.off[1], i[2] + Gf.off[2]);
        xf[fi] = __dadd_rn(xf[fi], __dmul_rn(sc, xc[gidx(Gc, I[0] + Gc.off[0], I[1] + Gc.off[1], I[2] + Gc.off[2])]));
    }
}

}  // namespace sw
