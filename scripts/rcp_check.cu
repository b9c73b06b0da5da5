// Accuracy of the stage path's branch-free fp64 reciprocal (kernels.cu fast_rcp: MUFU seed + r (1 + e + e^2)) against
// the correctly rounded 1/x, in ulps, over random positive normal arguments spanning 2^-60 .. 2^60 (and the
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

__global__ void check(unsigned long long n, unsigned long long seed, unsigned long long* maxulp,
                      unsigned long long* nonexact) {
    unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
    unsigned long long worst = 0, ne = 0;
    for (; i < n; i += (unsigned long long)gridDim.x * blockDim.x) {
        unsigned long long z = seed + i * 0x9E3779B97F4A7C15ull;   // SplitMix64
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        const int ex = (int)((z >> 52) % 121) - 60;                 // exponent -60 .. 60
        const double m = 1.0 + (double)(z & ((1ull << 52) - 1)) * 0x1p-52;
        const double x = ldexp(m, ex);
        const double a = rcp3(x), b = __drcp_rn(x);
        const long long d = __double_as_longlong(a) - __double_as_longlong(b);
        const unsigned long long u = d < 0 ? -d : d;
        worst = u > worst ? u : worst;
        ne += u != 0;
    }
    atomicMax(maxulp, worst);
    atomicAdd(nonexact, ne);
}

int main() {
    unsigned long long *d, h[2];
    cudaMalloc(&d, 16);
    cudaMemset(d, 0, 16);
    const unsigned long long n = 1ull << 30;
    check<<<148 * 8, 256>>>(n, 12345, d, d + 1);
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("{\"samples\": %llu, \"max_ulp\": %llu, \"not_correctly_rounded\": %llu}\n", n, h[0], h[1]);
    return h[0] > 1;
}
