// Microbenchmark: latency of warp primitives in a dependent chain (cycles).
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(unsigned *out, int n, long long *cyc) {
    __shared__ double sm[64];
    const int lane = threadIdx.x & 31;
    unsigned x = lane;
    double d = lane;
    sm[lane] = lane;
    __syncwarp();
    long long c0 = clock64();
    for (int i = 0; i < n; i++) {
        if (OP == 0) { __syncwarp(); x += 1; }
        if (OP == 1) x = __reduce_max_sync(0xffffffffu, x) + lane;
        if (OP == 2) x = __ballot_sync(0xffffffffu, x & 1) + lane;
        if (OP == 3) x = __shfl_sync(0xffffffffu, x, (x + 1) & 31);
        if (OP == 4) { d = sm[(int)d & 31] + 1.0; }
        if (OP == 5) { sm[lane] = d; __syncwarp(); d = sm[(lane + 1) & 31] + 1.0; }
    }
    long long c1 = clock64();
    out[lane] = x + (unsigned)d;
    if (lane == 0) cyc[0] = (c1 - c0) / n;
}
int main() {
    unsigned *out; long long *cyc, h;
    cudaMalloc(&out, 256); cudaMalloc(&cyc, 8);
    const char *names[] = {"__syncwarp", "__reduce_max_sync", "__ballot_sync", "__shfl_sync", "LDS chain", "STS+syncwarp+LDS"};
    k<0><<<1,32>>>(out, 4096, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("%s: %lld\n", names[0], h);
    k<1><<<1,32>>>(out, 4096, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("%s: %lld\n", names[1], h);
    k<2><<<1,32>>>(out, 4096, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("%s: %lld\n", names[2], h);
    k<3><<<1,32>>>(out, 4096, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("%s: %lld\n", names[3], h);
    k<4><<<1,32>>>(out, 4096, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("%s: %lld\n", names[4], h);
    k<5><<<1,32>>>(out, 4096, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("%s: %lld\n", names[5], h);
    return 0;
}
