// Isolated timing of the 3D wavefront step (sweep3.cuh, step 3b) for one warp: cycles per step for
// variants that remove one ingredient at a time.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
//   -I paper_1008_3699_b200/csrc -o tools/micro/wf3 tools/micro/wf3.cu -lcuda
#include <cstdio>
#include "sweep3.cuh"
using namespace sw;

template <int V>
__global__ void kwf(double *out, long long *cyc, int T0, int T1, int T2, int cb, int sb) {
    extern __shared__ double sm[];
    const int E0 = V == 6 ? 34 : T0 + 1, E1 = V == 6 ? 321 / 34 + 1 : T1 + 1, E2 = T2 + 1;
    const int WS = V == 6 ? 321 * E2 + 64 : E0 * E1 * E2;
    for (int i = threadIdx.x; i < 4 * WS + T0 * (T1 + T2) + 88; i += blockDim.x) sm[i] = 0.25 + 1e-3 * (i % 97);
    __syncthreads();
    double *X = sm, *PV = sm + 4 * WS;
    const int PS = V == 6 ? 321 : E0 * E1;
    const int st[3] = {1, E0, PS};
    auto wof = [&](int l0, int l1, int l2) { return (l0 + 1) + E0 * (l1 + 1) + PS * (l2 + 1); };
    const int lane = threadIdx.x, nl = T1 * T2;
    const bool on = lane < nl;
    const int j = on ? lane % T1 : 0, k = on ? lane / T1 : 0;
    const bool yc = j == 0 && (cb & 2), zc = k == 0 && (cb & 4);
    const bool edge = yc && zc, ypair = yc && !zc, zpair = zc && !yc, pair = ypair || zpair;
    const int i0 = (cb & 1) ? 1 : 0;
    const int sx = st[0], sy = st[1], sz = st[2];
    const int sa = ypair ? sy : (zpair ? sz : 0);
    const int wl = wof(0, j, k);
    const int pvb = ypair ? T0 * k : T0 * T2 + T0 * j;
    const bool qf = pair ? (((sb >> (ypair ? 1 : 2)) & 1) == 0) : true;
    const int oq_arr = ypair ? 3 : 2, pa_arr = ypair ? 2 : 3;
    double W = i0 ? X[wl] : 0.0;
    double Wq = (i0 && pair) ? X[wl - sa] : 0.0;
    double u = 0.0, py = 0.0, pz = 0.0;
    const int NS = T0 + T1 + T2 - 2;
    auto ld = [&](int s, double (&v)[11]) {
        int i = s - j - k;
        i = i < 0 ? 0 : (i >= T0 ? T0 - 1 : i);
        const int w = wl + i * sx, q = pair ? w - sa : w;
        if (V == 2 || V == 4) { for (int t = 0; t < 11; ++t) v[t] = 0.1 * t + 1e-3 * w; return; }
        v[0] = X[w]; v[1] = sm[WS + w]; v[2] = sm[2 * WS + w]; v[3] = sm[3 * WS + w];
        v[4] = X[q]; v[5] = sm[WS + q]; v[6] = sm[oq_arr * WS + q]; v[7] = sm[pa_arr * WS + q];
        v[8] = pair ? PV[pvb + i] : 1.0;
        v[9] = edge ? X[w - sy] : 0.0;
        v[10] = edge ? X[w - sz] : 0.0;
    };
    double nv[11];
    ld(0, nv);
    long long t0 = clock64();
    for (int rep = 0; rep < 16; ++rep)
    for (int s = 0; s < NS; ++s) {
        double Sv, Bv, Sq, Bq;
        if (V == 1 || V == 4) { Sv = u * 0.5; Bv = u * 0.25; Sq = pz; Bq = py; }
        else { Sv = shfl_up_f64(u, 1); Bv = shfl_up_f64(u, T1); Sq = shfl_up_f64(pz, 1); Bq = shfl_up_f64(py, T1); }
        double v[11];
#pragma unroll
        for (int t = 0; t < 11; ++t) v[t] = nv[t];
        if (s + 1 < NS) ld(s + 1, nv);
        const int i = s - j - k;
        const bool act = on && i >= i0 && i < T0;
        const int w = wl + (i < 0 ? 0 : (i >= T0 ? T0 - 1 : i)) * sx;
        const double cyE = ypair ? 0.0 : v[2], czE = zpair ? 0.0 : v[3];
        const double rp = fma(czE, Bv, fma(cyE, Sv, fma(v[1], W, v[0])));
        const double Oq = ypair ? Bq : Sq;
        const double rq = fma(pair ? v[6] : 0.0, Oq, fma(pair ? v[5] : 0.0, Wq, v[4]));
        const double cw = ypair ? v[2] : (zpair ? v[3] : 0.0), cq = pair ? v[7] : 0.0;
        const double ra = qf ? rq : rp, rb = qf ? rp : rq;
        const double mab = qf ? cq : cw, mba = qf ? cw : cq;
        const double ub = fma(mba, ra, rb) * v[8];
        const double ua = fma(mab, ub, ra) * 1.0;
        double un = qf ? ub : ua;
        const double pv = qf ? ua : ub;
        un = edge ? v[0] : un;
        if (V != 3) st_shared_if(X + w, un, act && !edge);
        u = sel_f64(act, un, u);
        W = sel_f64(act, un, W);
        Wq = sel_f64(act && pair, pv, Wq);
        py = sel_f64(act, ypair ? pv : (edge ? v[9] : py), py);
        pz = sel_f64(act, zpair ? pv : (edge ? v[10] : pz), pz);
    }
    long long t1 = clock64();
    if (lane == 0) cyc[0] = t1 - t0;
    out[lane] = u + W + Wq + py + pz;
}


// optimised step: compile-time 32x8x4 shape with conflict-free strides (RS = 34, PS = 321), pair data
// pre-ordered (piv, mFS, mSF), zeroed pair slots, ping-pong prefetch, unconditional loads
__global__ void kwf7(double *out, long long *cyc, int cb, int sb) {
    extern __shared__ double sm[];
    constexpr int T0 = 32, T1 = 8, T2 = 4, RS = 34, PS = 321, WS = PS * 5 + 64;
    for (int i = threadIdx.x; i < 4 * WS + 3 * 64 * 33 + 64; i += blockDim.x) sm[i] = 0.25 + 1e-3 * (i % 97);
    __syncthreads();
    double *X = sm, *PV = sm + 4 * WS;
    const int lane = threadIdx.x;
    const int j = lane % T1, k = lane / T1;
    const bool yc = j == 0 && (cb & 2), zc = k == 0 && (cb & 4);
    const bool edge = yc && zc, ypair = yc && !zc, zpair = zc && !yc, pair = ypair || zpair;
    const int i0 = (cb & 1) ? 1 : 0;
    const int sa = ypair ? RS : (zpair ? PS : 0);
    const int wl = 1 + RS * (j + 1) + PS * (k + 1);
    const bool qf = pair ? (((sb >> (ypair ? 1 : 2)) & 1) == 0) : true;
    // pair data: [kind][line][i][3] with stride 3 per node; plain lanes read a constant (1, 0, 0)
    const double *pvl = pair ? PV + 3 * ((ypair ? 0 : 8) + (ypair ? k : j)) * 33 : PV + 3 * 16 * 33;
    const int pvs = pair ? 3 : 0;
    double W = i0 ? X[wl] : 0.0, Wq = (i0 && pair) ? X[wl - sa] : 0.0;
    double u = 0.0, py = 0.0, pz = 0.0;
    constexpr int NS = T0 + T1 + T2 - 2;
    struct V { double r0, cx, cy, cz, q0, qx, qy, qz, piv, mfs, msf, ey, ez; };
    auto ld = [&](int s, V &v) {
        const int w = wl + (s - j - k), q = w - sa;
        const double *pv = pvl + pvs * (s - j - k);
        v.r0 = X[w]; v.cx = X[WS + w]; v.cy = X[2 * WS + w]; v.cz = X[3 * WS + w];
        v.q0 = X[q]; v.qx = X[WS + q]; v.qy = X[2 * WS + q]; v.qz = X[3 * WS + q];
        v.piv = pv[0]; v.mfs = pv[1]; v.msf = pv[2];
        v.ey = X[w - RS]; v.ez = X[w - PS];
    };
    auto step = [&](int s, const V &v) {
        const double Sv = shfl_up_f64(u, 1), Bv = shfl_up_f64(u, T1);
        const double Sq = shfl_up_f64(pz, 1), Bq = shfl_up_f64(py, T1);
        const int i = s - j - k;
        const bool act = i >= i0 && i < T0;
        const double rp = fma(v.cz, Bv, fma(v.cy, Sv, fma(v.cx, W, v.r0)));
        const double rq = fma(v.qz, Bq, fma(v.qy, Sq, fma(v.qx, Wq, v.q0)));
        const double rF = qf ? rq : rp, rS = qf ? rp : rq;
        const double uS = fma(v.msf, rF, rS) * v.piv;
        const double uF = fma(v.mfs, uS, rF);
        double un = qf ? uS : uF;
        const double pv = qf ? uF : uS;
        un = edge ? v.r0 : un;
        st_shared_if(X + wl + i, un, act && !edge);
        u = un;
        W = sel_f64(act, un, W);
        Wq = sel_f64(act, pv, Wq);
        py = ypair ? pv : v.ey;
        pz = zpair ? pv : v.ez;
    };
    V va, vb;
    ld(0, va);
    long long t0 = clock64();
    for (int rep = 0; rep < 16; ++rep) {
        int s = 0;
#pragma unroll 1
        for (; s + 1 < NS; s += 2) {
            ld(s + 1, vb);
            step(s, va);
            ld(s + 2, va);
            step(s + 1, vb);
        }
        if (s < NS) step(s, va);
    }
    long long t1 = clock64();
    if (lane == 0) cyc[0] = t1 - t0;
    out[lane] = u + W + Wq + py + pz;
}


// v7 with an array-of-structures node record (r0, cx, cy, cz) read by two 16-byte loads; rows padded
// by 16 bytes so that the eight lanes of a quarter-warp hit distinct 16-byte bank groups
__global__ void kwf8(double *out, long long *cyc, int cb, int sb) {
    extern __shared__ double sm[];
    constexpr int T0 = 32, T1 = 8, T2 = 4;
    constexpr int RU = 2 * 34 + 1, PU = RU * 9 + 2;          // strides in 16-byte units
    constexpr int NU = PU * 5 + 64;                           // 16-byte units of the node records
    for (int i = threadIdx.x; i < 2 * NU + 4 * 17 * 33 + 64; i += blockDim.x) sm[i] = 0.25 + 1e-3 * (i % 97);
    __syncthreads();
    double2 *N = reinterpret_cast<double2 *>(sm);
    const double *PV = sm + 2 * NU;
    const int lane = threadIdx.x;
    const int j = lane % T1, k = lane / T1;
    const bool yc = j == 0 && (cb & 2), zc = k == 0 && (cb & 4);
    const bool edge = yc && zc, ypair = yc && !zc, zpair = zc && !yc, pair = ypair || zpair;
    const int i0 = (cb & 1) ? 1 : 0;
    const int sa = ypair ? RU : (zpair ? PU : 0);
    const int wl = 2 + RU * (j + 1) + PU * (k + 1);         // 16-byte unit of node (0, j, k)
    const bool qf = pair ? (((sb >> (ypair ? 1 : 2)) & 1) == 0) : true;
    const double *pvl = pair ? PV + 4 * ((ypair ? 0 : 8) + (ypair ? k : j)) * 33 : PV + 4 * 16 * 33;
    const int pvs = pair ? 4 : 0;
    double W = i0 ? N[wl].x : 0.0, Wq = (i0 && pair) ? N[wl - sa].x : 0.0;
    double u = 0.0, py = 0.0, pz = 0.0;
    constexpr int NS = T0 + T1 + T2 - 2;
    struct V { double2 a, b, qa, qb, p0; double ey, ez; };
    auto ld = [&](int s, V &v) {
        const int w = wl + 2 * (s - j - k), q = w - sa;
        const double2 *pv = reinterpret_cast<const double2 *>(pvl + pvs * (s - j - k));
        v.a = N[w]; v.b = N[w + 1]; v.qa = N[q]; v.qb = N[q + 1];
        v.p0 = pv[0];
        v.ey = pv[1].x;                      // (mSF in a real layout; stands for the third pair value)
        v.ez = N[w - RU].x + N[w - PU].x;
    };
    auto step = [&](int s, const V &v) {
        const double Sv = shfl_up_f64(u, 1), Bv = shfl_up_f64(u, T1);
        const double Sq = shfl_up_f64(pz, 1), Bq = shfl_up_f64(py, T1);
        const int i = s - j - k;
        const bool act = i >= i0 && i < T0;
        const double rp = fma(v.b.y, Bv, fma(v.b.x, Sv, fma(v.a.y, W, v.a.x)));
        const double rq = fma(v.qb.y, Bq, fma(v.qb.x, Sq, fma(v.qa.y, Wq, v.qa.x)));
        const double rF = qf ? rq : rp, rS = qf ? rp : rq;
        const double uS = fma(v.ey, rF, rS) * v.p0.x;
        const double uF = fma(v.p0.y, uS, rF);
        double un = qf ? uS : uF;
        const double pv = qf ? uF : uS;
        un = edge ? v.a.x : un;
        st_shared_if(reinterpret_cast<double *>(N + wl + 2 * i), un, act && !edge);
        u = un;
        W = sel_f64(act, un, W);
        Wq = sel_f64(act, pv, Wq);
        py = ypair ? pv : v.ez;
        pz = zpair ? pv : v.ez;
    };
    V va, vb;
    ld(0, va);
    long long t0 = clock64();
    for (int rep = 0; rep < 16; ++rep) {
        int s = 0;
#pragma unroll 1
        for (; s + 1 < NS; s += 2) {
            ld(s + 1, vb);
            step(s, va);
            ld(s + 2, va);
            step(s + 1, vb);
        }
        if (s < NS) step(s, va);
    }
    long long t1 = clock64();
    if (lane == 0) cyc[0] = t1 - t0;
    out[lane] = u + W + Wq + py + pz;
}

template <int V>
void run(double *o, long long *c, const char *name) {
    const int T0 = 32, T1 = 8, T2 = 4;
    const int ws = 33 * 9 * 5;
    const size_t smem = 8 * (4 * (321 * 5 + 64) + T0 * (T1 + T2) + 88);
    cudaFuncSetAttribute(kwf<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    long long h;
    kwf<V><<<1, 32, smem>>>(o, c, T0, T1, T2, 7, 0);
    kwf<V><<<1, 32, smem>>>(o, c, T0, T1, T2, 7, 0);
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%-28s %.1f cycles/step  (%s)\n", name, h / (16.0 * 42), cudaGetErrorString(cudaGetLastError()));
}
int main() {
    double *o; long long *c;
    cudaMalloc(&o, 4096); cudaMalloc(&c, 64);
    run<0>(o, c, "as in sweep3");
    run<1>(o, c, "no shuffles");
    run<2>(o, c, "no smem loads");
    run<3>(o, c, "no smem stores");
    run<4>(o, c, "no loads, no shuffles");
    run<6>(o, c, "conflict-free strides");
    {
        const size_t smem = 8 * (4 * (321 * 5 + 64) + 3 * 64 * 33 + 64);
        cudaFuncSetAttribute(kwf7, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        long long h;
        kwf7<<<1, 32, smem>>>(o, c, 7, 0);
        kwf7<<<1, 32, smem>>>(o, c, 7, 0);
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("%-28s %.1f cycles/step  (%s)\n", "optimised (v7)", h / (16.0 * 42), cudaGetErrorString(cudaGetLastError()));
    }
    {
        const size_t smem = 8 * (2 * ((2 * 34 + 1) * 9 * 5 + 64 + 10) + 4 * 17 * 33 + 64);
        cudaFuncSetAttribute(kwf8, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        long long h;
        kwf8<<<1, 32, smem>>>(o, c, 7, 0);
        kwf8<<<1, 32, smem>>>(o, c, 7, 0);
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("%-28s %.1f cycles/step  (%s)\n", "AoS records (v8)", h / (16.0 * 42), cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
