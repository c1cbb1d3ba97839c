// Microbenchmark: cycles per step of the supernodal TRSM block factorization
// (glu_snode.cu task_trsm) for one warp alone on an SM, and its pieces:
// a dependent chain of __ddiv_rn, of DMUL+DADD, and the shared-memory step.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -fmad=false trsm_step.cu -o trsm_step
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double msub(double t, double l, double u) { return __dsub_rn(t, __dmul_rn(l, u)); }

__global__ void k_div(double *out, double a, double b, int n, long long *cyc) {
    double x = a == 0.0 ? (threadIdx.x == 0 ? 0.0 : 1.0 + threadIdx.x) : a + threadIdx.x;
    long long c0 = clock64();
    for (int i = 0; i < n; i++) x = __ddiv_rn(x, b);
    long long c1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = (c1 - c0) / n;
}
__global__ void k_mac(double *out, double a, double b, int n, long long *cyc) {
    double x = a + threadIdx.x;
    long long c0 = clock64();
    for (int i = 0; i < n; i++) x = msub(x, b, a);
    long long c1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = (c1 - c0) / n;
}
struct Sm { double b[16][33]; };
template <bool SAFE>
__global__ void k_block(double *out, int reps, int w, long long *cyc) {
    __shared__ Sm S;
    const int lane = threadIdx.x & 31;
    long long tot = 0;
    for (int r = 0; r < reps; r++) {
        for (int c = 0; c < 16; c++) S.b[c][lane] = (c == lane ? 4.0 + r : (lane < w ? 0.01 * (c + 1) * (lane + 1) : 0.0));
        __syncwarp();
        const int clol = 0;
        long long c0 = clock64();
        const bool inb = lane < w;
        unsigned long long bmax = 0;
        for (int j = 0; j < w; j++) {
            const unsigned has = __ballot_sync(0xffffffffu, clol <= j);
            const bool below = lane > j && inb;
            const double xj = S.b[j][lane];
            const unsigned long long m = __reduce_max_sync(0xffffffffu, below ? (unsigned)(__double_as_longlong(fabs(xj)) >> 32) : 0u);
            if (lane == j) bmax = m;
            const double piv = S.b[j][j];
            const double l = __ddiv_rn(SAFE ? (below ? xj : piv) : xj, piv);
            __syncwarp();
            if (below) {
                S.b[j][lane] = l;
#pragma unroll 4
                for (int c = j + 1; c < w; c++)
                    if ((has >> c) & 1u) S.b[c][lane] = msub(S.b[c][lane], l, S.b[c][j]);
            }
            __syncwarp();
        }
        tot += clock64() - c0;
        out[lane] += S.b[w - 1][lane] + (double)bmax;
    }
    if (lane == 0) cyc[0] = tot / reps / w;
}

int main() {
    double *out;
    long long *cyc, h;
    cudaMalloc(&out, 64 * sizeof(double));
    cudaMemset(out, 0, 64 * sizeof(double));
    cudaMalloc(&cyc, sizeof(long long));
    k_div<<<1, 32>>>(out, 1.7, 1.0000001, 4096, cyc);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("ddiv_rn dependent chain: %lld cycles\n", h);
    k_mac<<<1, 32>>>(out, 1.7, 0.999, 4096, cyc);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("DMUL+DADD dependent chain: %lld cycles per MAC\n", h);
    for (int w : {2, 8, 16}) {
        k_block<false><<<1, 32>>>(out, 200, w, cyc);
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("TRSM block step (w=%d): %lld cycles per step\n", w, h);
        k_block<true><<<1, 32>>>(out, 200, w, cyc);
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("TRSM block step, idle lanes divide piv/piv (w=%d): %lld cycles per step\n", w, h);
    }
    k_div<<<1, 32>>>(out, -0.0 * 1.7, 1.0000001, 4096, cyc);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("ddiv_rn of zero numerators (lane 0: 0/b, others lane/b): %lld cycles\n", h);
    return 0;
}
