// Microbenchmark: cost of publishing a task's stores (cycles per release):
// __threadfence (fence.sc.gpu) + atomicAdd, fence.acq_rel.gpu + red, and
// red.release.gpu, after 16 stores per lane, one warp per SM on every SM.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(double *buf, unsigned *cnt, int n, long long *cyc) {
    const int lane = threadIdx.x & 31;
    double *b = buf + (size_t)blockIdx.x * 4096;
    long long c0 = clock64();
    for (int i = 0; i < n; i++) {
        for (int s = 0; s < 16; s++) __stcg(b + s * 32 + lane, (double)(i + s));
        __syncwarp();
        if (lane == 0) {
            if (MODE == 0) { __threadfence(); atomicAdd(cnt + blockIdx.x * 32, 1u); }
            if (MODE == 1) { asm volatile("fence.acq_rel.gpu;" ::: "memory"); atomicAdd(cnt + blockIdx.x * 32, 1u); }
            if (MODE == 2) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" :: "l"(cnt + blockIdx.x * 32) : "memory");
        }
        __syncwarp();
    }
    long long c1 = clock64();
    if (lane == 0 && blockIdx.x == 0) cyc[0] = (c1 - c0) / n;
}
int main() {
    double *buf; unsigned *cnt; long long *cyc, h;
    cudaMalloc(&buf, 148ull * 4096 * 8); cudaMalloc(&cnt, 148 * 32 * 4); cudaMalloc(&cyc, 8);
    const char *nm[] = {"__threadfence + atomicAdd", "fence.acq_rel.gpu + atomicAdd", "red.release.gpu"};
    for (int rep = 0; rep < 2; rep++) {
        k<0><<<148, 32>>>(buf, cnt, 2000, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("%s: %lld cycles\n", nm[0], h);
        k<1><<<148, 32>>>(buf, cnt, 2000, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("%s: %lld cycles\n", nm[1], h);
        k<2><<<148, 32>>>(buf, cnt, 2000, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("%s: %lld cycles\n", nm[2], h);
    }
    return 0;
}
