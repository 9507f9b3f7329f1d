// mg.cuh -- grid transfer kernels of the geometric multigrid preconditioner:
// piecewise-constant aggregation of 2^d fine nodes into one coarse node, R = P^T, and the Galerkin
// coarse operator R A P, which is again a face-coefficient operator: each coarse face is the sum
// of the 2^(d-1) fine faces it covers, beta_c = 2^d beta (DESIGN R-19).  All sums in a fixed order
// (the lower index of the first remaining axis first, pairwise), mirrored by the oracle-side test.
#pragma once
#include "common.cuh"
#include "blas.cuh"

namespace sw {

// coarse face along axis a at coarse node I (I_a in [0, nc_a], the other axes in [0, nc_b))
template <int DIM>
__global__ void k_coarsen_faces(Geo Gf, Geo Gc, int a, const double *__restrict__ Ff, double *__restrict__ Fc) {
    int64_t m[3] = {1, 1, 1};
    for (int b = 0; b < DIM; ++b) m[b] = Gc.n[b] + (b == a ? 1 : 0);
    const int64_t total = m[0] * m[1] * m[2];
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t I[3] = {e % m[0], (e / m[0]) % m[1], e / (m[0] * m[1])};
        int64_t f[3] = {2 * I[0], 2 * I[1], 2 * I[2]};
        double v;
        auto F = [&](int64_t f0, int64_t f1, int64_t f2) {
            return Ff ? Ff[gidx(Gf, f0 + Gf.off[0], f1 + Gf.off[1], f2 + Gf.off[2])] : 1.0;
        };
        if (DIM == 1) {
            v = F(f[0], 0, 0);
        } else if (DIM == 2) {
            const int b = a == 0 ? 1 : 0;                 // the other axis
            int64_t g1[3] = {f[0], f[1], 0};
            g1[b] += 1;
            v = F(f[0], f[1], 0) + F(g1[0], g1[1], 0);
        } else {
            const int b = a == 0 ? 1 : 0, c = a == 2 ? 1 : 2;   // the other two axes, ascending
            int64_t q[4][3];
            for (int t = 0; t < 4; ++t) {
                q[t][0] = f[0]; q[t][1] = f[1]; q[t][2] = f[2];
                q[t][b] += t & 1;
                q[t][c] += t >> 1;
            }
            v = (F(q[0][0], q[0][1], q[0][2]) + F(q[1][0], q[1][1], q[1][2])) +
                (F(q[2][0], q[2][1], q[2][2]) + F(q[3][0], q[3][1], q[3][2]));
        }
        Fc[gidx(Gc, I[0] + Gc.off[0], I[1] + Gc.off[1], I[2] + Gc.off[2])] = v;
    }
}

// r_c[I] = sum of r over the 2^d fine nodes of I: pairs along x, then pairs of pairs along y, z
template <int DIM>
__global__ void k_restrict(Geo Gf, Geo Gc, const double *__restrict__ rf, double *__restrict__ rc) {
    const int64_t total = Gc.n[0] * Gc.n[1] * Gc.n[2];
    const int64_t S1 = Gf.P0, S2 = Gf.P01;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t I[3] = {e % Gc.n[0], (e / Gc.n[0]) % Gc.n[1], e / (Gc.n[0] * Gc.n[1])};
        const int64_t i = gidx(Gf, 2 * I[0] + Gf.off[0], 2 * I[1] + Gf.off[1], 2 * I[2] + Gf.off[2]);
        double v = rf[i] + rf[i + 1];
        if (DIM > 1) v = v + (rf[i + S1] + rf[i + S1 + 1]);
        if (DIM > 2) v = v + ((rf[i + S2] + rf[i + S2 + 1]) + (rf[i + S2 + S1] + rf[i + S2 + S1 + 1]));
        rc[gidx(Gc, I[0] + Gc.off[0], I[1] + Gc.off[1], I[2] + Gc.off[2])] = v;
    }
}

// r_c[I] = sum over the 2^d fine nodes of I of (r - A x), in k_restrict's order: the residual of
// the pre-smoothed iterate restricted in one pass (each fine residual as k_resid_r computes it)
template <int DIM, bool FACES>
__global__ void k_resid_restrict(Geo Gf, Geo Gc, double beta, const double *__restrict__ F0,
                                 const double *__restrict__ F1, const double *__restrict__ F2,
                                 const double *__restrict__ x, const double *__restrict__ r, double *__restrict__ rc) {
    const int64_t total = Gc.n[0] * Gc.n[1] * Gc.n[2];
    const int64_t S1 = Gf.P0, S2 = Gf.P01;
    auto res = [&](int64_t i) { return __dsub_rn(r[i], apply_A_fast<DIM, FACES>(F0, F1, F2, x, i, S1, S2, beta)); };
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t I[3] = {e % Gc.n[0], (e / Gc.n[0]) % Gc.n[1], e / (Gc.n[0] * Gc.n[1])};
        const int64_t i = gidx(Gf, 2 * I[0] + Gf.off[0], 2 * I[1] + Gf.off[1], 2 * I[2] + Gf.off[2]);
        double v = res(i) + res(i + 1);
        if (DIM > 1) v = v + (res(i + S1) + res(i + S1 + 1));
        if (DIM > 2) v = v + ((res(i + S2) + res(i + S2 + 1)) + (res(i + S2 + S1) + res(i + S2 + S1 + 1)));
        rc[gidx(Gc, I[0] + Gc.off[0], I[1] + Gc.off[1], I[2] + Gc.off[2])] = v;
    }
}

// x[i] += s x_c[i / 2]  (product and sum rounded separately; s = 1 adds x_c)
template <int DIM>
__global__ void k_prolong_add(Geo Gf, Geo Gc, double sc, const double *__restrict__ xc, double *__restrict__ xf) {
    const int64_t total = Gf.n[0] * Gf.n[1] * Gf.n[2];
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i[3] = {e % Gf.n[0], (e / Gf.n[0]) % Gf.n[1], e / (Gf.n[0] * Gf.n[1])};
        const int64_t fi = gidx(Gf, i[0] + Gf.off[0], i[1] + Gf.off[1], i[2] + Gf.off[2]);
        xf[fi] = __dadd_rn(xf[fi], __dmul_rn(sc, xc[gidx(Gc, i[0] / 2 + Gc.off[0], i[1] / 2 + Gc.off[1], i[2] / 2 + Gc.off[2])]));
    }
}

}  // namespace sw
