// Latency microbenchmarks on one B200 (diagnostics for the factor kernel design).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }

__global__ void chase(const int *next, int steps, int start, long long *out, int mode) {
    int p = start;
    long long t0 = clock64();
    for (int i = 0; i < steps; i++) {
        if (mode == 0) p = __ldcg(next + p);
        else { int x; asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(x) : "l"(next + p)); p = x; }
    }
    long long t1 = clock64();
    out[0] = (t1 - t0);
    out[1] = p;
}

__global__ void ddiv_chain(double *x, int steps, long long *out) {
    double a = x[0], b = x[1];
    long long t0 = clock64();
    for (int i = 0; i < steps; i++) a = __ddiv_rn(a, b) + 1.0;
    long long t1 = clock64();
    out[0] = t1 - t0; x[2] = a;
}
__global__ void dadd_chain(double *x, int steps, long long *out) {
    double a = x[0], b = x[1];
    long long t0 = clock64();
    for (int i = 0; i < steps; i++) a = __dsub_rn(a, b);
    long long t1 = clock64();
    out[0] = t1 - t0; x[2] = a;
}

// ping-pong between block 0 and block 1 (different SMs): flag[0], flag[1]
__global__ void pingpong(unsigned *flag, int rounds, long long *out, int use_red) {
    unsigned *mine = flag + (blockIdx.x ? 64 : 0), *other = flag + (blockIdx.x ? 0 : 64);
    if (threadIdx.x) return;
    unsigned long long t0 = gt();
    for (int r = 0; r < rounds; r++) {
        if (blockIdx.x == 0) {
            if (use_red) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" :: "l"(other) : "memory");
            else asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(other), "r"(r + 1) : "memory");
            unsigned v; do { asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(mine) : "memory"); } while (v < (unsigned)(r + 1));
        } else {
            unsigned v; do { asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(mine) : "memory"); } while (v < (unsigned)(r + 1));
            if (use_red) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" :: "l"(other) : "memory");
            else asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(other), "r"(r + 1) : "memory");
        }
    }
    unsigned long long t1 = gt();
    if (blockIdx.x == 0) out[0] = (long long)(t1 - t0);
}

__global__ void sleeper(long long *out, int ns) {
    unsigned long long t0 = gt();
    for (int i = 0; i < 1000; i++) __nanosleep(ns);
    out[0] = (long long)(gt() - t0);
}

// store then fence latency
__global__ void st_fence(double *x, int rounds, long long *out) {
    long long t0 = clock64();
    for (int i = 0; i < rounds; i++) { __stcg(x + i * 32, (double)i); asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
    long long t1 = clock64();
    out[0] = t1 - t0;
}

int main() {
    cudaSetDevice(0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double ghz = clk / 1e6;
    printf("sm clock attr %.3f GHz\n", ghz);
    long long *dout; cudaMalloc(&dout, 64); long long h[4];
    for (size_t mb : {4ul, 32ul, 64ul, 256ul, 2048ul}) {
        size_t n = mb * (1 << 20) / 4;
        std::vector<int> perm(n / 16);
        for (size_t i = 0; i < perm.size(); i++) perm[i] = (int)(i * 16);
        std::mt19937 rng(1); std::shuffle(perm.begin(), perm.end(), rng);
        std::vector<int> next(n, 0);
        for (size_t i = 0; i < perm.size(); i++) next[perm[i]] = perm[(i + 1) % perm.size()];
        int *d; cudaMalloc(&d, n * 4); cudaMemcpy(d, next.data(), n * 4, cudaMemcpyHostToDevice);
        for (int mode = 0; mode < 2; mode++) {
            chase<<<1, 1>>>(d, 20000, perm[0], dout, mode);  // warm
            chase<<<1, 1>>>(d, 20000, perm[0], dout, mode);
            cudaMemcpy(h, dout, 16, cudaMemcpyDeviceToHost);
            printf("chase %5zu MB mode %d: %.1f cycles/load = %.1f ns\n", mb, mode, h[0] / 20000.0, h[0] / 20000.0 / ghz);
        }
        cudaFree(d);
    }
    double *x; cudaMalloc(&x, 1 << 20); double hx[3] = {1.5, 1.0000001, 0};
    cudaMemcpy(x, hx, 24, cudaMemcpyHostToDevice);
    ddiv_chain<<<1, 1>>>(x, 10000, dout); cudaMemcpy(h, dout, 8, cudaMemcpyDeviceToHost);
    printf("ddiv+dadd chain: %.1f cycles/step\n", h[0] / 10000.0);
    dadd_chain<<<1, 1>>>(x, 10000, dout); cudaMemcpy(h, dout, 8, cudaMemcpyDeviceToHost);
    printf("dsub chain: %.1f cycles/step\n", h[0] / 10000.0);
    unsigned *flag; cudaMalloc(&flag, 4096);
    for (int red = 0; red < 2; red++) {
        cudaMemset(flag, 0, 4096);
        pingpong<<<2, 32>>>(flag, 10000, dout, red); cudaMemcpy(h, dout, 8, cudaMemcpyDeviceToHost);
        printf("pingpong (%s): %.1f ns per one-way handoff\n", red ? "red.release" : "st.release", h[0] / 20000.0);
    }
    for (int ns : {0, 32, 100, 500}) {
        sleeper<<<1, 32>>>(dout, ns); cudaMemcpy(h, dout, 8, cudaMemcpyDeviceToHost);
        printf("nanosleep(%d): %.1f ns each\n", ns, h[0] / 1000.0);
    }
    st_fence<<<1, 1>>>(x, 1000, dout); cudaMemcpy(h, dout, 8, cudaMemcpyDeviceToHost);
    printf("stcg + fence.acq_rel.gpu: %.1f cycles\n", h[0] / 1000.0);
    printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
