// Single-warp issue-rate microbenchmarks on B200: how many cycles one warp needs per instruction
// class when the instructions are independent (8 chains).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double *out, long long *cyc, double a, int n, int sel) {
    __shared__ double sm[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = i * 1e-3;
    __syncthreads();
    double x[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = threadIdx.x * 1e-3 + c;
    const bool p = (threadIdx.x & 1) != 0;
    long long t0, t1;
    // 8 independent DFMA chains
    t0 = clock64();
    for (int i = 0; i < n; ++i)
#pragma unroll
        for (int c = 0; c < 8; ++c) x[c] = fma(a, x[c], 1.0);
    t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
    // 8 independent double selects (runtime predicate)
    double y[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) y[c] = c * 0.5;
    t0 = clock64();
    for (int i = 0; i < n; ++i) {
        const bool q = p ^ (i & 1);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            y[c] = q ? x[c] + y[c] : y[c] - x[c];
        }
    }
    t1 = clock64();
    if (threadIdx.x == 0) cyc[1] = t1 - t0;
    // 8 independent LDS.64 per iteration (address depends on i)
    double acc = 0.0;
    t0 = clock64();
    for (int i = 0; i < n; ++i) {
        double v[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) v[c] = sm[((i * 37 + c * 33 + threadIdx.x * 9) & 2047)];
#pragma unroll
        for (int c = 0; c < 8; ++c) acc += v[c];
    }
    t1 = clock64();
    if (threadIdx.x == 0) cyc[2] = t1 - t0;
    // 8 SHFL.64 independent per iteration
    t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int c = 0; c < 8; ++c) y[c] = __shfl_up_sync(0xffffffffu, y[c], 1 + c);
    }
    t1 = clock64();
    if (threadIdx.x == 0) cyc[3] = t1 - t0;
    double s = acc;
#pragma unroll
    for (int c = 0; c < 8; ++c) s += x[c] + y[c];
    out[threadIdx.x] = s;
}
int main() {
    double *o; long long *c, h[8];
    cudaMalloc(&o, 8192); cudaMalloc(&c, 64);
    int n = 1024;
    for (int w = 1; w <= 4; w *= 2) {
        k<<<1, 32 * w>>>(o, c, 0.999, n, 0);
        cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
        printf("warps=%d per instruction (8 indep): DFMA %.2f  SELP.f64 %.2f  LDS.64(+DADD) %.2f  SHFL.64 %.2f cycles\n", w,
               h[0] / (8.0 * n), h[1] / (8.0 * n), h[2] / (8.0 * n), h[3] / (8.0 * n));
    }
    return 0;
}
