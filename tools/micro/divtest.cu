// Does the branch-free Newton/Markstein division equal IEEE n/d bitwise?  Random n in (0,2),
// d over many binades, plus the reciprocal-then-multiply variants.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ double rcp_approx(double d) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
    return r;
}
__device__ __forceinline__ double div_fast(double n, double d) {
    double y = rcp_approx(d);
    double e = fma(-d, y, 1.0);
    y = fma(y, e, y);
    e = fma(-d, y, 1.0);
    y = fma(y, e, y);
    double q = n * y;
    double r = fma(-d, q, n);
    return fma(r, y, q);
}
__device__ uint64_t mix(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__global__ void k(unsigned long long *bad, long long n, int mode) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        uint64_t a = mix(2 * i + mode * 0x12345), b = mix(2 * i + 1 + mode * 0x12345);
        double u = (a >> 11) * (1.0 / 9007199254740992.0), v = (b >> 11) * (1.0 / 9007199254740992.0);
        double nn = 2.0 * u + 1e-300;                  // (0, 2)
        double d = exp2(40.0 * v - 20.0);              // 2^-20 .. 2^20
        if (mode == 1) nn = 1.0;
        double q1 = nn / d, q2 = div_fast(nn, d);
        if (__double_as_longlong(q1) != __double_as_longlong(q2)) atomicAdd(bad, 1ull);
    }
}
int main() {
    unsigned long long *bad, h;
    cudaMalloc(&bad, 8);
    for (int mode = 0; mode < 2; ++mode) {
        cudaMemset(bad, 0, 8);
        long long n = 1ll << 32;
        k<<<148 * 16, 256>>>(bad, n, mode);
        cudaMemcpy(&h, bad, 8, cudaMemcpyDeviceToHost);
        printf("mode %d: %lld samples, %llu mismatches\n", mode, n, h);
    }
    return 0;
}
