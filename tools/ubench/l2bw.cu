// Microbenchmark: L2 read bandwidth (GB/s) -- a 64 MiB buffer (fits the
// 126 MB L2) read repeatedly by every SM with 16-byte ld.global.cg, after a
// warm-up pass.  The roofline denominator for L2-resident value traffic.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void rd(const double2 *__restrict__ p, size_t n, int reps, double *out) {
    double s = 0.0;
    for (int r = 0; r < reps; r++)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
            const double2 v = __ldcg(p + i);
            s += v.x + v.y;
        }
    if (s == 12345.678) out[0] = s;
}
int main() {
    const size_t bytes = 64ull << 20, n = bytes / 16;
    double2 *p; double *o;
    cudaMalloc(&p, bytes); cudaMalloc(&o, 8); cudaMemset(p, 0, bytes);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    rd<<<sms * 4, 512>>>(p, n, 1, o);
    for (int reps : {10, 40}) {
        cudaEventRecord(a);
        rd<<<sms * 4, 512>>>(p, n, reps, o);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("{\"l2_read_gbs\": %.1f, \"buffer_mib\": 64, \"reps\": %d, \"ms\": %.3f}\n", bytes * reps / (ms * 1e-3) / 1e9, reps, ms);
    }
    return 0;
}
