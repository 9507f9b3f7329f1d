// Latency microbenchmarks on B200: dependent DFMA, DADD, SHFL(64-bit), LDS/STS round trip, FSEL.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double *out, long long *cyc, double a, int n) {
    double x = threadIdx.x * 1e-3, y = 1.0;
    long long t0, t1;
    __shared__ double sm[64];
    sm[threadIdx.x] = x;
    __syncwarp();
    // DFMA chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = fma(a, x, y);
    t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
    // SHFL chain (64-bit)
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = __shfl_up_sync(0xffffffffu, x, 1) + 1.0;
    t1 = clock64();
    if (threadIdx.x == 0) cyc[1] = t1 - t0;
    // SHFL + DFMA (wavefront step)
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = fma(a, __shfl_up_sync(0xffffffffu, x, 1), y);
    t1 = clock64();
    if (threadIdx.x == 0) cyc[2] = t1 - t0;
    // STS -> LDS round trip
    volatile double *vs = sm;
    t0 = clock64();
    for (int i = 0; i < n; ++i) { vs[threadIdx.x] = x; x = vs[threadIdx.x] + 1.0; }
    t1 = clock64();
    if (threadIdx.x == 0) cyc[3] = t1 - t0;
    // DADD chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = x + a;
    t1 = clock64();
    if (threadIdx.x == 0) cyc[4] = t1 - t0;
    // DMUL chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = x * a;
    t1 = clock64();
    if (threadIdx.x == 0) cyc[5] = t1 - t0;
    out[threadIdx.x] = x;
}
int main() {
    double *o; long long *c, h[8];
    cudaMalloc(&o, 1024); cudaMalloc(&c, 64);
    int n = 4096;
    for (int w = 1; w <= 8; w *= 2) {
        k<<<1, 32 * w>>>(o, c, 0.999, n);
        cudaMemcpy(h, c, 48, cudaMemcpyDeviceToHost);
        printf("warps=%d  DFMA %.1f  SHFL64+DADD %.1f  SHFL64+DFMA %.1f  STS->LDS+DADD %.1f  DADD %.1f  DMUL %.1f cycles/iter\n", w,
               h[0] / (double)n, h[1] / (double)n, h[2] / (double)n, h[3] / (double)n, h[4] / (double)n, h[5] / (double)n);
    }
    // throughput: many independent warps of DFMA chains across the chip
    return 0;
}
