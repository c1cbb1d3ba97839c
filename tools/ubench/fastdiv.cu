// Checks the TRSM row division x / piv computed from a precomputed
// correctly rounded reciprocal r = RN(1 / piv) (two Markstein corrections)
// against __ddiv_rn, bit for bit, over random operand pairs.
//   q0 = RN(x r); e0 = RN(x - piv q0); q1 = RN(q0 + e0 r);
//   e1 = x - piv q1 (exact: q1 is faithful); q = RN(q1 + e1 r)
// Markstein's theorem: q is RN(x / piv) when q1 is a faithful quotient and r
// approximates 1/piv with relative error < 2^-53, barring under/overflow --
// the kernel takes this path only for |x| in [2^-400, 2^400] and |piv| in
// [2^-500, 2^500].  nvcc -O3 -gencode arch=compute_100a,code=sm_100a fastdiv.cu -o fastdiv
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ double fast_div(double x, double piv, double r) {
    const double q0 = __dmul_rn(x, r);
    const double e0 = __fma_rn(-piv, q0, x);
    const double q1 = __fma_rn(e0, r, q0);
    const double e1 = __fma_rn(-piv, q1, x);
    return __fma_rn(e1, r, q1);
}
__device__ __forceinline__ uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
__device__ double make(uint64_t bits, int emin, int emax) {
    const uint64_t m = bits & ((1ull << 52) - 1);
    const int e = emin + (int)((bits >> 52) % (uint64_t)(emax - emin + 1));
    const uint64_t s = (bits >> 63) << 63;
    return __longlong_as_double((long long)(s | ((uint64_t)(e + 1023) << 52) | m));
}
__global__ void check(uint64_t seed, uint64_t n, int mode, unsigned long long *bad, double *ex) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t a = mix(seed + 2 * i), b = mix(seed + 2 * i + 1);
        double x, piv;
        if (mode == 0) {  // random mantissas, the whole guarded range
            x = make(a, -400, 400);
            piv = make(b, -500, 500);
        } else if (mode == 1) {  // matrix-like magnitudes
            x = make(a, -60, 60);
            piv = make(b, -60, 60);
        } else if (mode == 3) {  // quotients next to a midpoint: x = RN(piv (q + ulp(q) / 2)) +- 1 ulp
            piv = make(b, -30, 30);
            const double q = make(a, -30, 30);
            const double hu = __longlong_as_double(__double_as_longlong(fabs(q)) & 0x7ff0000000000000ll) * 0x1p-53;
            const double p = __fma_rn(piv, q, __dmul_rn(piv, q < 0 ? -hu : hu));
            x = __longlong_as_double(__double_as_longlong(p) + (long long)((a >> 60) & 3) - 1);
        } else {  // quotients next to a representable number: x = piv * q with q's low bits random, perturbed by 1 ulp
            piv = make(b, -30, 30);
            const double q = make(a, -30, 30);
            const double p = __dmul_rn(piv, q);
            x = __longlong_as_double(__double_as_longlong(p) + (long long)((a >> 60) & 3) - 1);
        }
        const double r = __drcp_rn(piv);
        const double q = fast_div(x, piv, r), ref = __ddiv_rn(x, piv);
        if (__double_as_longlong(q) != __double_as_longlong(ref)) {
            const unsigned long long k = atomicAdd(bad, 1ull);
            if (k < 4) {
                ex[3 * k] = x;
                ex[3 * k + 1] = piv;
                ex[3 * k + 2] = q;
            }
        }
    }
}
int main(int argc, char **argv) {
    const int reps = argc > 1 ? atoi(argv[1]) : 8;
    unsigned long long *bad;
    double *ex;
    cudaMallocManaged(&bad, 8);
    cudaMallocManaged(&ex, 12 * 8);
    const uint64_t n = 1ull << 32;
    for (int mode = 0; mode < 4; mode++) {
        *bad = 0;
        for (int r = 0; r < reps; r++) check<<<148 * 8, 256>>>(0x9e3779b97f4a7c15ull * (r + 1) + mode * 0x1234567ull * n, n, mode, bad, ex);
        cudaDeviceSynchronize();
        printf("{\"mode\": %d, \"pairs\": %llu, \"mismatches\": %llu}\n", mode, (unsigned long long)n * reps, *bad);
        for (unsigned long long k = 0; k < *bad && k < 4; k++) printf("  x=%a piv=%a got=%a\n", ex[3 * k], ex[3 * k + 1], ex[3 * k + 2]);
    }
    return cudaGetLastError() != cudaSuccess;
}
