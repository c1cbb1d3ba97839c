// fence cost vs outstanding scattered stores (diagnostics)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void fence_cost(double *v, int nst, int stride, int rounds, long long *out, int busy) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (w > 0) {  // neighbour warps: keep loading from L2 (polling-like) if busy
        if (!busy) return;
        double acc = 0;
        for (int i = 0; i < rounds * 20; i++) acc += __ldcg(v + ((i * 977 + w * 131 + lane * 7) & ((1 << 22) - 1)));
        if (acc == 1.2345) out[3] = 1;
        return;
    }
    long long tot = 0;
    for (int r = 0; r < rounds; r++) {
        for (int s = 0; s < nst; s++) __stcg(v + (((size_t)(r * nst + s) * 32 + lane) * stride & ((1 << 22) - 1)), (double)r);
        __syncwarp();
        long long t0 = clock64();
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        long long t1 = clock64();
        tot += t1 - t0;
    }
    if (lane == 0) out[0] = tot / rounds;
}
int main() {
    double *v; cudaMalloc(&v, 8 << 22); long long *o; cudaMalloc(&o, 64); long long h;
    for (int busy = 0; busy < 2; busy++)
    for (int nst : {0, 1, 4, 16})
    for (int stride : {1, 37}) {
        fence_cost<<<1, busy ? 512 : 32>>>(v, nst, stride, 200, o, busy);
        cudaMemcpy(&h, o, 8, cudaMemcpyDeviceToHost);
        printf("busy=%d stores/lane=%2d stride=%2d: fence %lld cycles\n", busy, nst, stride, h);
    }
    // whole GPU busy: 148 blocks
    fence_cost<<<148, 512>>>(v, 4, 37, 200, o, 1); cudaMemcpy(&h, o, 8, cudaMemcpyDeviceToHost);
    printf("148 SMs busy, 4 stores/lane stride 37: fence %lld cycles\n", h);
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
