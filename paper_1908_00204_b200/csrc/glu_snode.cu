// glu_snode.cu -- supernodal engine: one persistent kernel over the phase-
// ordered warp tasks of glu_snode.cpp, then a pivot-check pass.
//
// Every task is one warp.  Warps walk the task list with a static stride
// (task i -> CTA i % grid, warp (i / grid) % 8, so consecutive tasks land on
// different SMs); a warp entering phase p waits until every task of phase
// p-1 has been counted, and counts its own tasks of a phase with one fence +
// one atomic when it leaves that phase.  Tasks of a phase only wait on
// smaller task indices, each warp runs its tasks in index order and all CTAs
// are co-resident (cooperative launch), so the walk cannot deadlock.
//
// Arithmetic is the reference's, bit for bit (levlu/_kernels.py:37-76,
// contract A): every MAC is __dsub_rn(t, __dmul_rn(Ldiv, U)) with the
// divided L value and the final U value, every divide __ddiv_rn, and every
// target receives its sources in ascending column order (panels in
// ascending order across stages, panel columns in ascending order inside a
// task's chain).  The pivot test |piv| <= thresh * max|column| runs after
// the factorization from per-column maxima gathered on the way (the
// undivided L values, the final U values), so a failing column is found
// exactly as the reference finds it; the columns after it are garbage, as
// the reference never computes them.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <string>
#include <vector>

#include "glu_b200.h"
#include "glu_internal.h"

using i64 = int64_t;
using i32 = int32_t;

namespace glu {

namespace {

constexpr int kSnThreads = 256;
constexpr int kSnWarps = kSnThreads / 32;
constexpr int kDoneStride = 8;  // u32 words between phase counters
constexpr unsigned long long kSnWatchdogNs = 4000000000ull;

struct SnParams {
    double *v;
    const i32 *col_ptr, *diag_pos, *col_a, *fail_level;
    const int4 *sn, *pan, *pairs, *push, *tasks;
    const i32 *relmap, *phase_ptr;
    i32 n_tasks;
    unsigned *done;
    unsigned long long *cmax;
    int *err;
};

__device__ __forceinline__ double ldv(const double *p) { return __ldcg(p); }
__device__ __forceinline__ void stv(double *p, double x) { __stcg(p, x); }
__device__ __forceinline__ double msub(double t, double l, double u) {
    return __dsub_rn(t, __dmul_rn(l, u));
}
// |x| as ordered bits (NaN ignored, like `av > cmax` in _kernels.py:61-64)
__device__ __forceinline__ unsigned long long absbits(double x) {
    const double a = fabs(x);
    return a == a ? (unsigned long long)__double_as_longlong(a) : 0ull;
}
__device__ __forceinline__ unsigned long long warp_max(unsigned long long m) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long y = __shfl_xor_sync(0xffffffffu, m, o);
        m = y > m ? y : m;
    }
    return m;
}
__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

struct WarpSmem {
    double b[kSnW][kSnW + 1];  // panel block, column-major [column][row]
    int clo[kSnW];             // per panel column: first panel row present
};

// first panel row present in column p0 + c (U rows of a supernode are a suffix)
__device__ __forceinline__ int panel_clo(const SnParams &P, int p0, int c) {
    return max(__ldg(P.col_a + p0 + c) - p0, 0);
}

// DIAG: column maxima above the block, then the w x w block factored in
// shared memory: step j divides column j below the diagonal and updates
// every later column (lanes = rows), each element receiving j ascending.
__device__ void task_diag(const SnParams &P, WarpSmem &S, int pi, int lane) {
    const int4 pn = __ldg(P.pan + pi);
    const int p0 = pn.x, w = pn.y - pn.x;
    unsigned long long mymax = 0;
    for (int c = 0; c < w; c++) {
        const int dc = __ldg(P.diag_pos + p0 + c);
        const int clo = panel_clo(P, p0, c);
        if (lane == 0) S.clo[c] = clo;
        const int pre_end = dc - (c - clo);
        unsigned long long m = 0;
        for (int q = __ldg(P.col_ptr + p0 + c) + lane; q < pre_end; q += 32) {
            const unsigned long long b = absbits(ldv(P.v + q));
            m = b > m ? b : m;
        }
        m = warp_max(m);
        if (lane == c) mymax = m;
        if (lane < w && lane >= clo) S.b[c][lane] = ldv(P.v + dc + (lane - c));
    }
    __syncwarp();
    for (int j = 0; j < w; j++) {
        const int cj = S.clo[j];
        const unsigned long long m = warp_max(lane < w && lane >= cj ? absbits(S.b[j][lane]) : 0ull);
        if (lane == j) mymax = m > mymax ? m : mymax;
        const double piv = S.b[j][j];
        if (lane > j && lane < w) S.b[j][lane] = __ddiv_rn(S.b[j][lane], piv);
        __syncwarp();
        if (lane > j && lane < w) {
            const double l = S.b[j][lane];
            for (int c = j + 1; c < w; c++)
                if (j >= S.clo[c]) S.b[c][lane] = msub(S.b[c][lane], l, S.b[c][j]);
        }
        __syncwarp();
    }
    for (int c = 0; c < w; c++) {
        const int clo = S.clo[c];
        if (lane < w && lane >= clo) stv(P.v + __ldg(P.diag_pos + p0 + c) + (lane - c), S.b[c][lane]);
    }
    if (lane < w) atomicMax(P.cmax + p0 + lane, mymax);
    __syncwarp();
}

// TRSM: 32 rows below the panel; lane = row, the row's w values in
// registers; step j takes the undivided value's maximum, divides, and
// updates the later columns with U(j, c) from the factored block.
__device__ void task_trsm(const SnParams &P, WarpSmem &S, int pi, int chunk, int lane) {
    const int4 pn = __ldg(P.pan + pi);
    const int p0 = pn.x, p1 = pn.y, w = p1 - p0, h = pn.w;
    for (int c = 0; c < w; c++) {
        const int dc = __ldg(P.diag_pos + p0 + c);
        const int clo = panel_clo(P, p0, c);
        if (lane == 0) S.clo[c] = clo;
        if (lane <= c && lane >= clo) S.b[c][lane] = ldv(P.v + dc + (lane - c));
    }
    __syncwarp();
    const int t = chunk * 32 + lane;
    const bool act = t < h;
    double x[kSnW];
#pragma unroll
    for (int c = 0; c < kSnW; c++)
        x[c] = (act && c < w) ? ldv(P.v + __ldg(P.diag_pos + p0 + c) + (p1 - p0 - c) + t) : 0.0;
    unsigned long long mymax = 0;
#pragma unroll
    for (int j = 0; j < kSnW; j++) {
        if (j < w) {
            const unsigned long long m = warp_max(act ? absbits(x[j]) : 0ull);
            if (lane == j) mymax = m;
            const double d = __ddiv_rn(x[j], S.b[j][j]);
            x[j] = d;
#pragma unroll
            for (int c = j + 1; c < kSnW; c++)
                if (c < w && j >= S.clo[c]) x[c] = msub(x[c], d, S.b[c][j]);
        }
    }
    if (act) {
#pragma unroll
        for (int c = 0; c < kSnW; c++)
            if (c < w) stv(P.v + __ldg(P.diag_pos + p0 + c) + (p1 - p0 - c) + t, x[c]);
    }
    if (lane < w) atomicMax(P.cmax + p0 + lane, mymax);
    __syncwarp();
}

// TRI: U(P, k) for every target column k of the push (lane = column):
// forward substitution with the panel's unit-lower block, j ascending.
__device__ void task_tri(const SnParams &P, WarpSmem &S, int xi, int lane) {
    const int4 ps = __ldg(P.push + xi);
    const int4 pn = __ldg(P.pan + ps.x);
    const int p0 = pn.x, p1 = pn.y, w = p1 - p0;
    const int s1 = __ldg(P.sn + pn.z).y;
    for (int j = 0; j < w; j++)
        if (lane > j && lane < w) S.b[j][lane] = ldv(P.v + __ldg(P.diag_pos + p0 + j) + (lane - j));
    __syncwarp();
    const int q = ps.y + lane;
    int4 pr = make_int4(0, p1, 0, -1);
    if (q < ps.z) pr = __ldg(P.pairs + q);
    const bool act = pr.y < p1;
    const int lo = max(pr.y - p0, 0);
    double u[kSnW];
#pragma unroll
    for (int r = 0; r < kSnW; r++)
        u[r] = (act && r < w && r >= lo) ? ldv(P.v + pr.z - (s1 - (p0 + r))) : 0.0;
#pragma unroll
    for (int j = 0; j < kSnW; j++) {
        if (j < w && act && j >= lo) {
            const double uj = u[j];
#pragma unroll
            for (int r = j + 1; r < kSnW; r++)
                if (r < w) u[r] = msub(u[r], S.b[j][r], uj);
        }
    }
    if (act) {
#pragma unroll
        for (int r = 0; r < kSnW; r++)
            if (r < w && r > lo) stv(P.v + pr.z - (s1 - (p0 + r)), u[r]);
    }
    __syncwarp();
}

// RECT: 32 rows below the source panel into every target column of the
// push: lane = row, its divided L row in registers, U(j, k) broadcast by
// shuffle, the chain over j ascending.
__device__ void task_rect(const SnParams &P, int xi, int chunk, int lane) {
    const int4 ps = __ldg(P.push + xi);
    const int4 pn = __ldg(P.pan + ps.x);
    const int p0 = pn.x, p1 = pn.y, w = p1 - p0, h = pn.w;
    const int4 sn = __ldg(P.sn + pn.z);
    const int s1 = sn.y, in_sn = s1 - p1;
    const int t = chunk * 32 + lane;
    const bool act = t < h;
    double L[kSnW];
#pragma unroll
    for (int j = 0; j < kSnW; j++)
        L[j] = (act && j < w) ? ldv(P.v + __ldg(P.diag_pos + p0 + j) + (p1 - p0 - j) + t) : 0.0;
    for (int q = ps.y; q < ps.z; q++) {
        const int4 pr = __ldg(P.pairs + q);
        if (pr.y >= p1) continue;
        const int lo = max(pr.y - p0, 0);
        const double uval = (lane < w && lane >= lo) ? ldv(P.v + pr.z - (s1 - (p0 + lane))) : 0.0;
        int pos = 0;
        if (act) {
            if (t < in_sn) pos = pr.z - (in_sn - t);
            else pos = pr.w >= 0 ? __ldg(P.relmap + pr.w + (t - in_sn)) : pr.z + (t - in_sn);
        }
        double x = act ? ldv(P.v + pos) : 0.0;
#pragma unroll
        for (int j = 0; j < kSnW; j++) {
            if (j < w && j >= lo) {
                const double uj = __shfl_sync(0xffffffffu, uval, j);
                x = msub(x, L[j], uj);
            }
        }
        if (act) stv(P.v + pos, x);
    }
}

__global__ void __launch_bounds__(kSnThreads, 2) sn_kernel(SnParams P) {
    extern __shared__ __align__(16) unsigned char sn_smem_raw[];
    WarpSmem *smem = reinterpret_cast<WarpSmem *>(sn_smem_raw);
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    WarpSmem &S = smem[wib];
    const int nw = gridDim.x * kSnWarps;
    int cur = -1;
    unsigned mine = 0;
    for (int i = wib * gridDim.x + blockIdx.x; i < P.n_tasks; i += nw) {
        const int4 tk = __ldg(P.tasks + i);
        if (tk.w != cur) {
            if (mine) {
                __syncwarp();
                if (lane == 0) {
                    __threadfence();
                    atomicAdd(P.done + (size_t)cur * kDoneStride, mine);
                }
            }
            mine = 0;
            cur = tk.w;
            if (cur > 0) {
                bool bail = false;
                if (lane == 0) {
                    const unsigned need = (unsigned)(__ldg(P.phase_ptr + cur) - __ldg(P.phase_ptr + cur - 1));
                    const unsigned *ctr = P.done + (size_t)(cur - 1) * kDoneStride;
                    if (ld_acquire(ctr) < need) {
                        const unsigned long long t0 = globaltimer();
                        while (ld_acquire(ctr) < need) {
                            if (*(volatile int *)P.err) { bail = true; break; }
                            __nanosleep(64);
                            if (globaltimer() - t0 > kSnWatchdogNs) {
                                atomicExch(P.err, 1);
                                bail = true;
                                break;
                            }
                        }
                    }
                }
                if (__shfl_sync(0xffffffffu, (int)bail, 0)) return;
            }
        }
        switch (tk.z) {
            case kSnDiag: task_diag(P, S, tk.x, lane); break;
            case kSnTrsm: task_trsm(P, S, tk.x, tk.y, lane); break;
            case kSnTri: task_tri(P, S, tk.x, lane); break;
            default: task_rect(P, tk.x, tk.y, lane); break;
        }
        mine++;
    }
    if (mine) {
        __syncwarp();
        if (lane == 0) {
            __threadfence();
            atomicAdd(P.done + (size_t)cur * kDoneStride, mine);
        }
    }
}

// pivot test of every column (_kernels.py:60-65): |piv| <= thresh * cmax
__global__ void sn_check_kernel(const double *v, const i32 *diag_pos, const unsigned long long *cmax,
                                const i32 *fail_level, i32 n, double thresh, int by_column,
                                unsigned long long *fail) {
    for (i32 c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
        const double piv = __ldcg(v + diag_pos[c]);
        const double cm = __longlong_as_double((long long)cmax[c]);
        if (fabs(piv) <= __dmul_rn(thresh, cm)) {
            const unsigned long long key =
                by_column ? (unsigned long long)c
                          : (((unsigned long long)__ldg(fail_level + c)) << 32) | (unsigned)c;
            atomicMin(fail, key);
        }
    }
}

template <class T>
cudaError_t up(T **dst, const std::vector<T> &src, i64 *bytes) {
    *dst = nullptr;
    if (src.empty()) return cudaSuccess;
    cudaError_t e = cudaMalloc((void **)dst, src.size() * sizeof(T));
    if (e != cudaSuccess) return e;
    *bytes += (i64)(src.size() * sizeof(T));
    return cudaMemcpy(*dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice);
}

}  // namespace

struct SnDev {
    int4 *sn = nullptr, *pan = nullptr, *pairs = nullptr, *push = nullptr, *tasks = nullptr;
    i32 *relmap = nullptr, *phase_ptr = nullptr, *col_a = nullptr;
    i64 n = 0, n_tasks = 0, n_phases = 0;
    unsigned *done = nullptr;
    unsigned long long *cmax = nullptr;
    int grid = 0;
};

constexpr size_t kSnSmem = sizeof(WarpSmem) * kSnWarps;

int sn_grid(int sm_count) {
    int per_sm = 0;
    if (cudaFuncSetAttribute(sn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSnSmem) != cudaSuccess)
        return 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sn_kernel, kSnThreads, kSnSmem) != cudaSuccess)
        return 0;
    return per_sm * sm_count;
}

void sn_free(SnDev *d) {
    if (!d) return;
    void *ptrs[] = {d->sn, d->pan, d->pairs, d->push, d->tasks, d->relmap, d->phase_ptr, d->col_a,
                    d->done, d->cmax};
    for (void *p : ptrs)
        if (p) cudaFree(p);
    delete d;
}

int64_t sn_upload(const SnPlan *p, SnDev **out, int64_t *bytes) {
    *out = nullptr;
    auto *d = new SnDev();
    auto cast = [](const std::vector<I4> &v) -> const std::vector<int4> & {
        return reinterpret_cast<const std::vector<int4> &>(v);
    };
    static_assert(sizeof(I4) == sizeof(int4), "I4 layout");
    cudaError_t e = cudaSuccess;
    if (e == cudaSuccess) e = up(&d->sn, cast(p->sn), bytes);
    if (e == cudaSuccess) e = up(&d->pan, cast(p->pan), bytes);
    if (e == cudaSuccess) e = up(&d->pairs, cast(p->pairs), bytes);
    if (e == cudaSuccess) e = up(&d->push, cast(p->push), bytes);
    if (e == cudaSuccess) e = up(&d->tasks, cast(p->tasks), bytes);
    if (e == cudaSuccess) e = up(&d->relmap, p->relmap, bytes);
    if (e == cudaSuccess) e = up(&d->phase_ptr, p->phase_ptr, bytes);
    if (e == cudaSuccess) e = up(&d->col_a, p->col_a, bytes);
    d->n = p->n;
    d->n_tasks = (i64)p->tasks.size();
    d->n_phases = (i64)p->phase_ptr.size() - 1;
    if (e == cudaSuccess)
        e = cudaMalloc((void **)&d->done, sizeof(unsigned) * kDoneStride * std::max<i64>(d->n_phases, 1));
    if (e == cudaSuccess) e = cudaMalloc((void **)&d->cmax, sizeof(unsigned long long) * std::max<i64>(d->n, 1));
    if (e != cudaSuccess) {
        set_error(std::string("supernodal plan upload: ") + cudaGetErrorString(e));
        sn_free(d);
        return GLU_ECUDA;
    }
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    d->grid = sn_grid(sms);
    if (d->grid <= 0) {
        set_error("supernodal kernel cannot be co-resident");
        sn_free(d);
        return GLU_ECUDA;
    }
    *out = d;
    return GLU_OK;
}

int64_t sn_launch(SnDev *d, double *v, const int32_t *col_ptr, const int32_t *diag_pos,
                  const int32_t *fail_level, int32_t n, double thresh, bool by_column,
                  unsigned long long *fail, int *err, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(d->done, 0, sizeof(unsigned) * kDoneStride * std::max<i64>(d->n_phases, 1), s);
    if (e == cudaSuccess) e = cudaMemsetAsync(d->cmax, 0, sizeof(unsigned long long) * std::max<i64>(d->n, 1), s);
    if (e == cudaSuccess) e = cudaMemsetAsync(err, 0, sizeof(int), s);
    if (e != cudaSuccess) {
        set_error(std::string("sn_launch: ") + cudaGetErrorString(e));
        return GLU_ECUDA;
    }
    if (d->n_tasks > 0) {
        SnParams P;
        P.v = v;
        P.col_ptr = col_ptr;
        P.diag_pos = diag_pos;
        P.col_a = d->col_a;
        P.fail_level = fail_level;
        P.sn = d->sn;
        P.pan = d->pan;
        P.pairs = d->pairs;
        P.push = d->push;
        P.tasks = d->tasks;
        P.relmap = d->relmap;
        P.phase_ptr = d->phase_ptr;
        P.n_tasks = (i32)d->n_tasks;
        P.done = d->done;
        P.cmax = d->cmax;
        P.err = err;
        void *args[] = {&P};
        e = cudaLaunchCooperativeKernel((const void *)sn_kernel, dim3(d->grid), dim3(kSnThreads), args, kSnSmem, s);
        if (e != cudaSuccess) {
            set_error(std::string("sn_kernel: ") + cudaGetErrorString(e));
            return GLU_ECUDA;
        }
    }
    if (n > 0) {
        sn_check_kernel<<<std::min<i64>((n + 255) / 256, 1184), 256, 0, s>>>(v, diag_pos, d->cmax, fail_level, n,
                                                                            thresh, by_column ? 1 : 0, fail);
        e = cudaGetLastError();
        if (e != cudaSuccess) {
            set_error(std::string("sn_check_kernel: ") + cudaGetErrorString(e));
            return GLU_ECUDA;
        }
    }
    return GLU_OK;
}

}  // namespace glu
