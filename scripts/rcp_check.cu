// Accuracy of the stage path's branch-free fp64 reciprocal (kernels.cu fast_rcp: MUFU seed + r (1 + e + e^2)) against
// the correctly rounded 1/x, and of fast_rsqrt / fast_sqrt (x / sqrt(x)) against the correctly rounded sqrt, in ulps, over random positive normal arguments spanning 2^-60 .. 2^60 (and the
// scheme's typical 0.01 .. 100).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/rcp_check
// scripts/rcp_check.cu
#include <cstdio>
#include <cstdint>
#include <cmath>

__device__ __forceinline__ double rcp3(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);
    e = fma(e, e, e);
    return fma(r, e, r);
}

__device__ __forceinline__ double rsqrt_poly(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double t = fma(x * y, y, -1.0);
    return fma(y, t * fma(0.375, t, -0.5), y);
}

__device__ __forceinline__ unsigned long long ulps(double a, double b) {
    const long long d = __double_as_longlong(a) - __double_as_longlong(b);
    return d < 0 ? -d : d;
}

__global__ void check(unsigned long long n, unsigned long long seed, unsigned long long* maxulp,
                      unsigned long long* nonexact) {
    unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
    unsigned long long worst = 0, ne = 0, wsq = 0, wrs = 0;
    for (; i < n; i += (unsigned long long)gridDim.x * blockDim.x) {
        unsigned long long z = seed + i * 0x9E3779B97F4A7C15ull;   // SplitMix64
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        const int ex = (int)((z >> 52) % 121) - 60;                 // exponent -60 .. 60
        const double m = 1.0 + (double)(z & ((1ull << 52) - 1)) * 0x1p-52;
        const double x = ldexp(m, ex);
        const unsigned long long u = ulps(rcp3(x), __drcp_rn(x));
        worst = u > worst ? u : worst;
        ne += u != 0;
        const double rs = rsqrt_poly(x), sq = __dsqrt_rn(x);
        const unsigned long long us = ulps(x * rs, sq);                 // sqrt = x / sqrt(x) vs correctly rounded
        wsq = us > wsq ? us : wsq;
        // 1/sqrt against 1/s refined by one Newton step on s^2 = x (a reference within ~0.5 ulp)
        const double r0 = __drcp_rn(sq), ref = fma(r0, 0.5 * fma(-sq, sq, x) * __drcp_rn(x), r0);
        const unsigned long long ur = ulps(rs, ref);
        wrs = ur > wrs ? ur : wrs;
    }
    atomicMax(maxulp, worst);
    atomicAdd(nonexact, ne);
    atomicMax(maxulp + 2, wsq);
    atomicMax(maxulp + 3, wrs);
}

int main() {
    unsigned long long *d, h[4];
    cudaMalloc(&d, 32);
    cudaMemset(d, 0, 32);
    const unsigned long long n = 1ull << 30;
    check<<<148 * 8, 256>>>(n, 12345, d, d + 1);
    cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
    printf("{\"samples\": %llu, \"rcp_max_ulp\": %llu, \"rcp_not_correctly_rounded\": %llu, \"sqrt_max_ulp\": %llu, "
           "\"rsqrt_max_ulp\": %llu}\n", n, h[0], h[1], h[2], h[3]);
    return h[0] > 1 || h[2] > 2 || h[3] > 2;
}
