// Microbenchmark of the dense-tail panel step (tools/ubench/panel.cu):
// one warp factors a 16x16 block (lane i = row i): per step a shuffle of the
// pivot row, a correctly rounded divide and 15 independent multiply/subtract
// pairs; variants with and without the global store of the L value.
#include <cstdio>
#include <cuda_runtime.h>

template <bool STORE>
__global__ void block_steps(double *g, int reps, long long *out) {
    const int lane = threadIdx.x & 31;
    double r[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) r[k] = 1.0 + 0.001 * (lane * 16 + k) + (lane == k ? 16.0 : 0.0);
    long long t0 = clock64();
    for (int rep = 0; rep < reps; ++rep) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const double piv = __shfl_sync(0xffffffffu, r[k], k);
            const bool bi = lane > k && lane < 16;
            double l = 0.0;
            if (bi) {
                l = __ddiv_rn(r[k], piv);
                if (STORE) __stcg(g + k * 64 + lane, l);
            }
#pragma unroll
            for (int kk = k + 1; kk < 16; ++kk) {
                const double u = __shfl_sync(0xffffffffu, r[kk], k);
                r[kk] = __dsub_rn(r[kk], bi ? __dmul_rn(l, u) : 0.0);
            }
        }
#pragma unroll
        for (int k = 0; k < 16; ++k) r[k] = r[k] * 1e-3 + 1.0 + (lane == k ? 16.0 : 0.0);
    }
    long long t1 = clock64();
    if (lane == 0) out[0] = t1 - t0;
    double acc = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) acc += r[k];
    if (acc == 12345.0) g[lane] = acc;
}

// rows-below form: each thread, its own row, divisor/U from shared memory
__global__ void row_steps(double *g, int reps, long long *out) {
    __shared__ double ub[16 * 16];
    const int t = threadIdx.x;
    for (int e = t; e < 256; e += blockDim.x) ub[e] = 1.0 + 0.01 * e + ((e / 16) == (e % 16) ? 16.0 : 0.0);
    __syncthreads();
    double r[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) r[k] = 1.0 + 0.001 * (t + k);
    long long t0 = clock64();
    for (int rep = 0; rep < reps; ++rep) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const double l = __ddiv_rn(r[k], ub[k * 16 + k]);
#pragma unroll
            for (int kk = k + 1; kk < 16; ++kk) r[kk] = __dsub_rn(r[kk], __dmul_rn(l, ub[k * 16 + kk]));
        }
#pragma unroll
        for (int k = 0; k < 16; ++k) r[k] = r[k] * 1e-3 + 1.0;
    }
    long long t1 = clock64();
    if (t == 0) out[0] = t1 - t0;
    double acc = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) acc += r[k];
    if (acc == 12345.0) g[t] = acc;
}

int main() {
    double *g;
    long long *d, h;
    cudaMalloc(&g, 1 << 20);
    cudaMalloc(&d, 8);
    const int reps = 200;
    block_steps<false><<<1, 32>>>(g, reps, d);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("block step (1 warp, no store): %.0f cycles/step\n", h / (16.0 * reps));
    block_steps<true><<<1, 32>>>(g, reps, d);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("block step (1 warp, store):    %.0f cycles/step\n", h / (16.0 * reps));
    for (int th : {32, 128, 512}) {
        row_steps<<<1, th>>>(g, reps, d);
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("row step (%3d threads):        %.0f cycles/step\n", th, h / (16.0 * reps));
    }
    return 0;
}
