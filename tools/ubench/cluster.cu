// cluster barrier cost (diagnostics)
#include <cstdio>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
__global__ void cbar(int rounds, long long *out, double *g, int mode) {
    extern __shared__ double sm[];
    cg::cluster_group cl = cg::this_cluster();
    long long t0 = clock64();
    for (int r = 0; r < rounds; r++) {
        if (mode == 1 && cl.block_rank() == (r % cl.num_blocks())) {
            for (int i = threadIdx.x; i < 8192; i += blockDim.x) __stcg(g + i, (double)r);
        }
        if (mode == 2) { asm volatile("barrier.cluster.arrive.relaxed;" ::: "memory"); asm volatile("barrier.cluster.wait;" ::: "memory"); }
        else cl.sync();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[cl.block_rank()] = (t1 - t0) / rounds;
    sm[threadIdx.x] = 0;
}
int main() {
    long long *o; cudaMalloc(&o, 1024); double *g; cudaMalloc(&g, 1 << 20);
    cudaFuncSetAttribute(cbar, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(cbar, cudaFuncAttributeMaxDynamicSharedMemorySize, 229000);
    for (int C : {2, 8, 16})
    for (int threads : {128, 512})
    for (int mode : {0, 1, 2}) {
        cudaLaunchConfig_t cfg = {}; cudaLaunchAttribute a[1];
        a[0].id = cudaLaunchAttributeClusterDimension; a[0].val.clusterDim.x = C; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(C); cfg.blockDim = dim3(threads); cfg.dynamicSmemBytes = 229000; cfg.attrs = a; cfg.numAttrs = 1;
        cudaError_t e = cudaLaunchKernelEx(&cfg, cbar, 2000, o, g, mode);
        long long h[16]; cudaMemcpy(h, o, 8 * C, cudaMemcpyDeviceToHost);
        printf("C=%2d threads=%3d mode=%d (%s): %lld cycles/sync  [%s]\n", C, threads, mode, mode == 0 ? "cl.sync" : mode == 1 ? "cl.sync + 64KB global stores by one CTA" : "arrive.relaxed+wait", h[0], cudaGetErrorString(e));
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
