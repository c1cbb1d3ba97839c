// glu_snode.cu -- supernodal engine: one persistent dataflow kernel over the
// warp tasks of glu_snode.cpp, then a pivot-check pass.
//
// Every task is one warp.  Each warp walks its own list of tasks (built at
// upload, sn_assign: round-robin over the list, consecutive tasks on
// different SMs) in list order.  There is no phase and no grid barrier: a
// task waits only for the counters of what it reads (glu_snode.cpp step 6)
// --
//   TRSM(P)   in[P] == every RECT chunk of every push into P
//   RECT(x)   f[P] == every TRSM chunk of its source panel, then
//             in[K] == every RECT chunk of the earlier pushes into K
//   RG        in[K] once, then each push's f[P] as it reaches the push
//   UW(x)     in[K] == the RECT chunks of x as well
//   WB(P)     f[P] == every TRSM chunk of P (they read the unfactored block)
// -- and counts itself with one fence + one atomic when done.  Every
// dependency has a smaller list index, each warp runs its tasks in list
// order and all CTAs are co-resident (cooperative launch), so the walk
// cannot deadlock: the smallest unfinished task can always run.

// A RECT task loads everything that is final once its source panel is
// factored (its L rows, the factored diagonal block, the target positions)
// BEFORE it waits for its target panel, so the chain of pushes into one
// target panel -- the engine's critical path -- carries only the target
// loads, the FP64 chains and the release.
//
// Arithmetic is the reference's, bit for bit (levlu/_kernels.py:37-76,
// contract A): every MAC is __dsub_rn(t, __dmul_rn(Ldiv, U)) with the
// divided L value and the final U value, every divide __ddiv_rn, and every
// target receives its sources in ascending column order (pushes into a
// target panel in ascending source panel, panel columns in ascending order
// inside a task's chain).  The pivot test |piv| <= thresh * max|column| runs
// after the factorization from per-column maxima gathered on the way (the
// undivided L values, the final U values), so a failing column is found
// exactly as the reference finds it; the columns after it are garbage, as
// the reference never computes them.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <queue>
#include <thread>
#include <type_traits>
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
constexpr unsigned long long kSnWatchdogNs = 4000000000ull;
// diagnostics trace, per task: {start, source ready, target ready, done, warp,
// TRSM phase cycles}
constexpr int kTraceWords = 6;

struct SnParams {
    double *v;
    double *dblk;  // factored diagonal blocks of panels with w >= 2, column-major w x w
    const i32 *diag_pos, *col_a;
    const int4 *pairs, *tasks, *panm;  // tasks: 3 records each (glu_internal.h SnPlan::tasks)
    const int4 *push, *pan;            // RG tasks: push {panel, pair0, pair1, K}, panel {p0, p1, S, h}
    const i32 *rg_slot;
    const uint16_t *rg_idx, *rg_uidx;
    const i32 *relmap;
    i32 n_tasks;
    unsigned *cnt;  // per panel P: [2P] RECT chunks into P done, [2P + 1] TRSM chunks of P done
    unsigned *fin;  // per panel: WB / UW tasks done (its values final once panm.w are; host copy-out)
    unsigned long long *cmax;
    int *err;
    unsigned long long *trace;  // optional: per task kTraceWords words
    const int *wptr;            // per warp: its tasks [wptr[g], wptr[g + 1]) of the warp-major task array
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
// max over the warp of non-negative double bit patterns: (hi, lo) lexicographic
__device__ __forceinline__ unsigned long long warp_max(unsigned long long m) {
    const unsigned hi = (unsigned)(m >> 32);
    const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
    const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? (unsigned)m : 0u);
    return ((unsigned long long)mh << 32) | ml;
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
__device__ __forceinline__ unsigned ld_relaxed(const unsigned *p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Wait until *c >= need: lane 0 polls with relaxed loads (an acquire load
// invalidates the SM's L1 each time), backing off, then one acquire load
// once the count is reached; the warp barrier orders every lane's later
// loads after it.  False on the watchdog / error path.
__device__ __forceinline__ bool wait_ge(const SnParams &P, const unsigned *c, unsigned need, int lane) {
    int ok = 1;
    if (lane == 0 && need > 0 && ld_acquire(c) < need) {
        const unsigned long long t0 = globaltimer();
        unsigned ns = 16;
        while (ld_relaxed(c) < need || ld_acquire(c) < need) {
            if (*(volatile int *)P.err) { ok = 0; break; }
            if (globaltimer() - t0 > kSnWatchdogNs) {
                atomicExch(P.err, 1);
                ok = 0;
                break;
            }
            __nanosleep(ns);
            ns = ns < 128 ? 2 * ns : ns;
        }
    }
    __syncwarp();
    return __shfl_sync(0xffffffffu, ok, 0) != 0;
}

// Tasks with two waits (source, then target) poll both counters in one
// round -- lane 0 the first, lane 1 the second, acquire loads in parallel --
// and skip the wait of each count already reached: a task whose inputs are
// complete when its warp reaches it (most tasks behind a busy warp) saves
// the second L2 round trip.  Bit k: counter k reached.  The warp barrier
// orders every lane's later loads after the acquires.
__device__ __forceinline__ unsigned poll2(const unsigned *c0, unsigned n0, const unsigned *c1, unsigned n1,
                                          int lane) {
    bool ok = true;
    if (lane < 2) {
        const unsigned *c = lane ? c1 : c0;
        const unsigned n = lane ? n1 : n0;
        ok = n == 0 || ld_acquire(c) >= n;
    }
    __syncwarp();
    return __ballot_sync(0xffffffffu, ok) & 3u;
}

// x / piv correctly rounded (__ddiv_rn) for the lanes that need it (use):
// the others divide piv / piv, and a zero x gives the signed zero directly
// -- a zero numerator or an idle lane's garbage sends __ddiv_rn down its
// slow path (~430 vs ~125 cycles, tools/ubench/trsm_step.cu), which the
// whole warp then waits for.  0 / piv for finite non-zero piv is the zero
// with sign(x) xor sign(piv), exactly what __ddiv_rn returns.
__device__ __forceinline__ double div_rn(double x, double piv, bool use) {
    const bool z = x == 0.0 && piv != 0.0 && fabs(piv) <= 1.7976931348623157e308;
    const double q = __ddiv_rn(use && !z ? x : piv, piv);
    return z ? __longlong_as_double((__double_as_longlong(x) ^ __double_as_longlong(piv)) & (1ll << 63)) : q;
}

// 8-byte global -> shared copy, zero-filled when !valid.  Through L1
// (.ca): every task's loads follow its acquire, which invalidates the SM's
// L1, so no line older than the data the task waited for can be hit.
__device__ __forceinline__ void cp_async8(void *dst, const double *src, bool valid, const double *any) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(valid ? src : any), "r"(valid ? 8 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Count a finished task: every lane's stores, then (lane 0) a device-scope
// fence and the counter increment.
__device__ __forceinline__ void release(unsigned *c, int lane) {
    __syncwarp();
    if (lane == 0) {
        __threadfence();
        atomicAdd(c, 1u);
    }
}

constexpr int kB = 32;  // lanes: shared-memory tile dimension

// Per-warp shared memory.  The task code is kept compact on purpose --
// runtime loops over shared-memory tiles instead of fully unrolled register
// chains per panel width: the warps of an SM run different task kinds and
// widths side by side, and a kernel much larger than the 32 KB L1.5
// instruction cache stalls them on instruction fetch (a fully unrolled
// 16-wide TRSM alone is ~40 KB of SASS).
struct TrsmSmem {
    double b[kSnW][kB + 1];  // the diagonal block, column-major [column][row]
    double x[kSnW][kB];      // the chunk's rows below the panel, [column][row = lane]
    double u[kSnW][kB];      // their undivided values (the column maxima)
};
struct RectSmem {
    double l[kSnW][kB];     // [j][row]: divided L rows below the source panel
    double u[kSnW][kSnW];   // [j][target column]: U(P, K)
    double lb[kSnW][kSnW];  // [j][r]: L(r, j) of the factored diagonal block
    int lo[kSnW];           // per target column: first panel row present
};
struct RgSmem {
    double val[kRgSlots];      // the staged slots
    double L[kRgRows];         // the pushes' L rows, push after push
    uint16_t idx[kRgIdx];      // MAC -> slot index
    uint16_t uidx[kRgPushes * kSnW];  // (push, pair) -> index of U(p0, k)
};
union WarpSmem {
    TrsmSmem t;
    RectSmem r;
    RgSmem g;
};

// Panel metadata, lane = panel column: its diagonal slot and the first
// panel row present in it (a supernode's U rows in a column are a suffix).
__device__ __forceinline__ void panel_cols(const SnParams &P, int p0, int w, int lane, int &dc, int &clo) {
    dc = 0;
    clo = kB;
    if (lane < w) {
        dc = __ldg(P.diag_pos + p0 + lane);
        clo = max(__ldg(P.col_a + p0 + lane) - p0, 0);
    }
}

// Structural predicates that change stored values (a supernode's partial U
// suffix, col_a) are selects, never a subtraction of a zero product: x - l * 0
// is not always x (x = -0 with l < 0, or l = inf).

// TRSM(P, chunk), w >= 2: the w x w diagonal block is factored locally
// (every push into P is done, and nothing writes the block in place during
// the kernel: chunk 0 stores the factored block in the scratch area, written
// back after the kernel, and records the block's L-part column maxima), then
// the chunk's 32 rows below the panel.  Lane = row.  Block step j: every
// row r > j takes column j's undivided value (its maximum over the block's
// L part is column j's), divides it by the pivot and updates its later
// columns with U(j, c), so every element receives its sources j in
// ascending order.  Row step j: the same with the factored block.
__device__ void task_trsm(const SnParams &P, TrsmSmem &S, int4 ta, int4 tb, int4 pm, int lane,
                          unsigned long long *tr) {
    const long long c0 = clock64();
    const int chunk = ta.x & 0x07ffffff;
    const int p0 = ta.z, p1 = ta.w, w = p1 - p0, h = tb.y;
    int dcl, clol;
    panel_cols(P, p0, w, lane, dcl, clol);
    const int t = chunk * 32 + lane;
    const bool act = t < h;
    // the block and the rows, copied straight to shared memory (all in flight at once)
#pragma unroll 1
    for (int c = 0; c < w; c++) {
        const int dc = __shfl_sync(0xffffffffu, dcl, c), clo = __shfl_sync(0xffffffffu, clol, c);
        cp_async8(&S.b[c][lane], P.v + dc + (lane - c), lane < w && lane >= clo, P.v);
        cp_async8(&S.x[c][lane], P.v + dc + (w - c) + t, act, P.v);
    }
    cp_async_wait();
    __syncwarp();
    const long long c1 = clock64();
    const bool inb = lane < w;
    // two lanes per block row r = lane % 16: each takes every other column
    const int br = lane & (kSnW - 1), hf = lane >> 4;
    for (int j = 0; j < w; j++) {
        const unsigned has = __ballot_sync(0xffffffffu, clol <= j);  // bit c: U(j, c) present
        const bool below = br > j && br < w;
        const double xj = S.b[j][br];
        const double l = div_rn(xj, S.b[j][j], below);
        __syncwarp();
        if (below) {
            if (hf == 0) {
                S.b[j][br] = l;
                S.u[j][br] = xj;  // undivided, for the column maximum (taken after the loop)
            }
            // 4 of this lane's columns at a time: loads, chains, stores (row j is
            // never written in step j)
            for (int c = j + 1 + hf; c < w; c += 8) {
                double a[4], u[4];
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    const int ck = min(c + 2 * k, kSnW - 1);
                    a[k] = S.b[ck][br];
                    u[k] = S.b[ck][j];
                }
#pragma unroll
                for (int k = 0; k < 4; k++)
                    if (c + 2 * k < w && ((has >> (c + 2 * k)) & 1u)) S.b[c + 2 * k][br] = msub(a[k], l, u[k]);
            }
        }
        __syncwarp();
    }
    const long long c2 = clock64();
    if (chunk == 0) {
        // the block's L-part column maxima (rows below the diagonal, undivided)
        unsigned long long bmax = 0;
        for (int c = 0; c < w - 1; c++) {
            const unsigned long long m = warp_max(lane > c && lane < w ? absbits(S.u[c][lane]) : 0ull);
            if (lane == c) bmax = m;
        }
        if (inb && pm.z >= 0)
            for (int c = 0; c < w; c++) stv(P.dblk + pm.z + c * w + lane, S.b[c][lane]);
        if (inb && bmax) atomicMax(P.cmax + p0 + lane, bmax);
        __syncwarp();  // S.u is reused by the rows below
    }
    // the rows (a register version, steps unrolled over the class width,
    // measured 4x slower: 16 inlined divisions with their slow-path calls).
    // The next column's value is carried in a register from the step that
    // updates it, and the column maxima (of the undivided values) are taken
    // after the loop, off the step-to-step chain.
    double xn = S.x[0][lane];
    for (int j = 0; j < w; j++) {
        const unsigned has = __ballot_sync(0xffffffffu, clol <= j);
        const double xj = xn;
        S.u[j][lane] = xj;  // undivided, for the column maximum
        const double d = div_rn(xj, S.b[j][j], act);
        S.x[j][lane] = d;
        xn = j + 1 < w ? S.x[j + 1][lane] : 0.0;
        if (j + 1 < w && ((has >> (j + 1)) & 1u)) xn = msub(xn, d, S.b[j + 1][j]);
        for (int c = j + 2; c < w; c += 4) {
            double a[4], u[4];
#pragma unroll
            for (int k = 0; k < 4; k++) {
                const int ck = min(c + k, kSnW - 1);
                a[k] = S.x[ck][lane];
                u[k] = S.b[ck][j];
            }
#pragma unroll
            for (int k = 0; k < 4; k++)
                if (c + k < w && ((has >> (c + k)) & 1u)) S.x[c + k][lane] = msub(a[k], d, u[k]);
        }
    }
    for (int c = 0; c < w; c++) {
        const int dc = __shfl_sync(0xffffffffu, dcl, c);
        if (act) stv(P.v + dc + (w - c) + t, S.x[c][lane]);
    }
    __syncwarp();
    unsigned long long mymax = 0;
    for (int c = 0; c < w; c++) {
        const unsigned long long m = warp_max(act ? absbits(S.u[c][lane]) : 0ull);
        if (lane == c) mymax = m;
    }
    if (inb && mymax) atomicMax(P.cmax + p0 + lane, mymax);
    __syncwarp();
    if (tr && lane == 0) {  // diagnostics: SM cycles of the loads, the block, the rows (21 bits each)
        const long long c3 = clock64();
        auto f = [](long long x) { return (unsigned long long)min(max(x, 0ll), (1ll << 21) - 1); };
        tr[5] = f(c1 - c0) | f(c2 - c1) << 21 | f(c3 - c2) << 42;
    }
}

// TRSM for a one-column panel: divide the rows below by the pivot.
__device__ void task_trsm1(const SnParams &P, int4 ta, int4 tb, int lane) {
    const int chunk = ta.x & 0x07ffffff;
    const int p0 = ta.z, h = tb.y;
    const int t = chunk * 32 + lane;
    const int dc = __ldg(P.diag_pos + p0);
    const double x = t < h ? ldv(P.v + dc + 1 + t) : 0.0;
    const double piv = ldv(P.v + dc);
    const unsigned long long m = warp_max(t < h ? absbits(x) : 0ull);
    const double q = div_rn(x, piv, t < h);
    if (t < h) stv(P.v + dc + 1 + t, q);
    if (lane == 0 && m) atomicMax(P.cmax + p0, m);
}

// Target slot of source-panel row t (rows below p1, in_sn of them inside
// the supernode) in the column of pair {k, a, base, map}.
__device__ __forceinline__ int target_pos(const SnParams &P, int t, int in_sn, int base, int map) {
    return t < in_sn ? base - (in_sn - t) : (map >= 0 ? __ldg(P.relmap + map + (t - in_sn)) : base + (t - in_sn));
}

// RECT for a one-column source panel (most pushes): lane = row t, the
// target slots of every column of the push found before the target wait,
// then every target loaded at once, one MAC each with U(p0, k) (held by
// lane q, broadcast by shuffle).
__device__ bool task_rect1(const SnParams &P, int4 ta, int4 tb, int4 tc, int lane, unsigned long long *tr) {
    const int chunk = ta.x & 0x07ffffff;
    const int Pi = ta.y, p0 = ta.z, p1 = ta.w, h = tb.y;
    const int s1 = tb.x, in_sn = s1 - p1;
    const int t = chunk * 32 + lane;
    const bool act = t < h;
    const int npair = tb.w - tb.z;
    const int4 pm = __ldg(P.panm + Pi);
    int4 myp = make_int4(0, p1, 0, -1);
    if (lane < npair) myp = __ldg(P.pairs + tb.z + lane);
    const bool colok = lane < npair && myp.y < p1;
    const int dc = __ldg(P.diag_pos + p0);
    int pos[kSnW];
#pragma unroll
    for (int q = 0; q < kSnW; q++) {
        const int base = __shfl_sync(0xffffffffu, myp.z, q);
        const int map = __shfl_sync(0xffffffffu, myp.w, q);
        const bool ok = __shfl_sync(0xffffffffu, (int)colok, q) != 0;
        pos[q] = (ok && act) ? target_pos(P, t, in_sn, base, map) : -1;
    }
    const unsigned rdy = poll2(P.cnt + 2 * Pi + 1, (unsigned)pm.y, P.cnt + 2 * tc.x, (unsigned)tc.y, lane);
    if (!(rdy & 1) && !wait_ge(P, P.cnt + 2 * Pi + 1, (unsigned)pm.y, lane)) return false;
    if (tr && lane == 0) tr[1] = globaltimer();
    const double L = act ? ldv(P.v + dc + 1 + t) : 0.0;
    if (!(rdy & 2) && !wait_ge(P, P.cnt + 2 * tc.x, (unsigned)tc.y, lane)) return false;
    if (tr && lane == 0) tr[2] = globaltimer();
    const double u = colok ? ldv(P.v + myp.z - (s1 - p0)) : 0.0;  // U(p0, k_lane)
    double x[kSnW];
#pragma unroll
    for (int q = 0; q < kSnW; q++) x[q] = pos[q] >= 0 ? ldv(P.v + pos[q]) : 0.0;
#pragma unroll
    for (int q = 0; q < kSnW; q++) {
        const double uq = __shfl_sync(0xffffffffu, u, q);
        if (pos[q] >= 0) stv(P.v + pos[q], msub(x[q], L, uq));
    }
    return true;
}

// U(P, K) of a push in shared memory: lane q < 16 holds target column q
// (asynchronous copies: cp_async_wait + __syncwarp before use).
__device__ __forceinline__ void load_u_tile(const SnParams &P, RectSmem &R, int4 myp, bool colok, int mylo,
                                            int p0, int w, int s1, int lane) {
    if (lane < kSnW) {
        R.lo[lane] = mylo;
#pragma unroll 1
        for (int j = 0; j < w; j++)
            cp_async8(&R.u[j][lane], P.v + myp.z - (s1 - (p0 + j)), colok && j >= mylo, P.v);
    }
}
// The forward substitution U(r, k) -= L(r, j) * U(j, k), j ascending.
__device__ __forceinline__ void solve_u_tile(RectSmem &R, bool colok, int mylo, int w, int lane) {
    // Column q = lane % 16 lives in two lanes: half h = lane / 16 holds its
    // rows 2s + h (s < 8) in registers (a shared-memory chain would
    // serialize every step behind the previous store: ~10k cycles for w = 16;
    // one lane per column issues twice the FP64 instructions).  Step j takes
    // U(j, k) from the half that owns row j (a shuffle) and updates the rows
    // below it, so every element keeps its chain over j ascending.  Selects
    // keep absent U(j, k) (j < lo) out; rows >= w hold garbage that only
    // feeds rows below them, which are never read back for the product.
    const int q = lane & (kSnW - 1), h = lane >> 4;
    const bool act = __shfl_sync(0xffffffffu, (int)colok, q) != 0;
    const int qlo = __shfl_sync(0xffffffffu, mylo, q);
    const int lo = act ? qlo : 0;  // absent columns: never stored
    double u[kSnW / 2];
#pragma unroll
    for (int s = 0; s < kSnW / 2; s++) u[s] = R.u[2 * s + h][q];
#pragma unroll
    for (int j = 0; j < kSnW - 1; j++) {
        const int sj = j >> 1;
        const double uj = __shfl_sync(0xffffffffu, u[sj], q | (j & 1) << 4);
        if (j >= lo) {
            if ((j & 1) == 0) {  // row j = 2 sj sits in half 0: half 1's slot sj is row j + 1
                const double y = msub(u[sj], R.lb[j][2 * sj + h], uj);
                u[sj] = h ? y : u[sj];
            }
#pragma unroll
            for (int s = sj + 1; s < kSnW / 2; s++) u[s] = msub(u[s], R.lb[j][2 * s + h], uj);
        }
    }
    __syncwarp();
    if (act) {
#pragma unroll
        for (int s = 0; s < kSnW / 2; s++) R.u[2 * s + h][q] = u[s];
    }
}
__device__ __forceinline__ void load_lb(const SnParams &P, RectSmem &R, int off, int w, int lane) {
#pragma unroll 1
    for (int e = lane; e < w * w; e += 32) {
        const int j = e / w, r = e - j * w;
        cp_async8(&R.lb[j][r], P.dblk + off + e, true, P.v);
    }
}

// RECT for source panels with w >= 2: register-tiled block C[32 rows x 16
// target columns] -= L[32 x w] * U[w x 16], every element's chain over j
// ascending, after the forward substitution of U(P, K) inside the source
// block when the push changes it.  Lane (ry, cx) = (lane / 4, lane % 4)
// holds rows ry + 8 i and columns cx + 4 k (i, k < 4); per j it reads 4 L and
// 4 U values from shared memory (conflict-free broadcasts) for 16 MACs.
// Columns whose U suffix starts inside the panel (lo > 0, only in
// structurally unsymmetric patterns) take the select path.
__device__ bool task_rect(const SnParams &P, RectSmem &R, int4 ta, int4 tb, int4 tc, int lane,
                          unsigned long long *tr) {
    const int code = (int)((unsigned)ta.x >> 27);
    const int chunk = ta.x & 0x07ffffff;
    const int Pi = ta.y, p0 = ta.z, p1 = ta.w, w = p1 - p0, h = tb.y;
    const int s1 = tb.x, in_sn = s1 - p1;
    const int npair = tb.w - tb.z;
    const int t = chunk * 32 + lane;
    const int4 pm = __ldg(P.panm + Pi);
    int4 myp = make_int4(0, p1, 0, -1);
    if (lane < npair) myp = __ldg(P.pairs + tb.z + lane);
    const bool colok = lane < npair && myp.y < p1;
    const int mylo = colok ? max(myp.y - p0, 0) : kB;
    const int dcl = lane < w ? __ldg(P.diag_pos + p0 + lane) : 0;
    const int ry = lane >> 2, cx = lane & 3;
    int pos[4][4];
#pragma unroll
    for (int k = 0; k < 4; k++) {
        const int q = cx + 4 * k;
        const int base = __shfl_sync(0xffffffffu, myp.z, q), map = __shfl_sync(0xffffffffu, myp.w, q);
        const bool cok = __shfl_sync(0xffffffffu, (int)colok, q) != 0;
#pragma unroll
        for (int i = 0; i < 4; i++) {
            const int tt = chunk * 32 + ry + 8 * i;
            pos[i][k] = (cok && tt < h) ? target_pos(P, tt, in_sn, base, map) : -1;
        }
    }
    const unsigned rdy = poll2(P.cnt + 2 * Pi + 1, (unsigned)pm.y, P.cnt + 2 * tc.x, (unsigned)tc.y, lane);
    if (!(rdy & 1) && !wait_ge(P, P.cnt + 2 * Pi + 1, (unsigned)pm.y, lane)) return false;
    if (tr && lane == 0) tr[1] = globaltimer();
#pragma unroll 1
    for (int j = 0; j < w; j++) {
        const int dj = __shfl_sync(0xffffffffu, dcl, j);
        cp_async8(&R.l[j][lane], P.v + dj + (w - j) + t, t < h, P.v);
    }
    const bool tri = (code & kSnTriF) != 0;
    if (tri) load_lb(P, R, pm.z, w, lane);
    if (!(rdy & 2) && !wait_ge(P, P.cnt + 2 * tc.x, (unsigned)tc.y, lane)) return false;
    if (tr && lane == 0) tr[2] = globaltimer();
    const long long c0 = clock64();
    load_u_tile(P, R, myp, colok, mylo, p0, w, s1, lane);
    const bool anylo = __any_sync(0xffffffffu, colok && mylo > 0);
    double c[4][4];
#pragma unroll
    for (int k = 0; k < 4; k++)
#pragma unroll
        for (int i = 0; i < 4; i++) c[i][k] = pos[i][k] >= 0 ? ldv(P.v + pos[i][k]) : 0.0;
    cp_async_wait();  // L rows, the factored block, U(P, K)
    __syncwarp();
    const long long c1 = clock64();
    if (tri) {
        solve_u_tile(R, colok, mylo, w, lane);
        __syncwarp();
    }
    const long long c2 = clock64();
    if (!anylo) {  // every column's U suffix starts at the panel: no selects
#pragma unroll 2
        for (int j = 0; j < w; j++) {
            double l[4], u[4];
#pragma unroll
            for (int i = 0; i < 4; i++) l[i] = R.l[j][ry + 8 * i];
#pragma unroll
            for (int k = 0; k < 4; k++) u[k] = R.u[j][cx + 4 * k];
#pragma unroll
            for (int i = 0; i < 4; i++)
#pragma unroll
                for (int k = 0; k < 4; k++) c[i][k] = msub(c[i][k], l[i], u[k]);
        }
    } else {
        int clo[4];
#pragma unroll
        for (int k = 0; k < 4; k++) clo[k] = R.lo[cx + 4 * k];
#pragma unroll 1
        for (int j = 0; j < w; j++) {
            double l[4], u[4];
#pragma unroll
            for (int i = 0; i < 4; i++) l[i] = R.l[j][ry + 8 * i];
#pragma unroll
            for (int k = 0; k < 4; k++) u[k] = R.u[j][cx + 4 * k];
#pragma unroll
            for (int i = 0; i < 4; i++)
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    const double y = msub(c[i][k], l[i], u[k]);
                    c[i][k] = j >= clo[k] ? y : c[i][k];
                }
        }
    }
#pragma unroll
    for (int k = 0; k < 4; k++)
#pragma unroll
        for (int i = 0; i < 4; i++)
            if (pos[i][k] >= 0) stv(P.v + pos[i][k], c[i][k]);
    if ((code & kSnWriteU) && lane < kSnW && colok)
        for (int r = mylo + 1; r < w; r++) stv(P.v + myp.z - (s1 - (p0 + r)), R.u[r][lane]);
    __syncwarp();
    if (tr && lane == 0) {  // diagnostics: SM cycles of the loads, the U solve, the MACs + stores
        const long long c3 = clock64();
        auto f = [](long long x) { return (unsigned long long)min(max(x, 0ll), (1ll << 21) - 1); };
        tr[5] = f(c1 - c0) | f(c2 - c1) << 21 | f(c3 - c2) << 42;
    }
    return true;
}

// UW(x): after every RECT chunk of push x has read U(P, K), solve it once
// more (the same chains, so the same bits) and write it.
__device__ bool task_uw(const SnParams &P, RectSmem &R, int4 ta, int4 tb, int4 tc, int lane,
                        unsigned long long *tr) {
    const int Pi = ta.y, p0 = ta.z, p1 = ta.w, w = p1 - p0, s1 = tb.x;
    const int npair = tb.w - tb.z;
    const int4 pm = __ldg(P.panm + Pi);
    int4 myp = make_int4(0, p1, 0, -1);
    if (lane < npair) myp = __ldg(P.pairs + tb.z + lane);
    const bool colok = lane < npair && myp.y < p1;
    const int mylo = colok ? max(myp.y - p0, 0) : kB;
    // the RECT chunks waited for P's TRSM chunks (which wrote the block)
    if (!wait_ge(P, P.cnt + 2 * tc.x, (unsigned)(tc.y + pm.y), lane)) return false;
    if (tr && lane == 0) tr[1] = tr[2] = globaltimer();
    load_lb(P, R, pm.z, w, lane);
    load_u_tile(P, R, myp, colok, mylo, p0, w, s1, lane);
    cp_async_wait();
    __syncwarp();
    solve_u_tile(R, colok, mylo, w, lane);
    __syncwarp();
    if (lane < kSnW && colok)
        for (int r = mylo + 1; r < w; r++) stv(P.v + myp.z - (s1 - (p0 + r)), R.u[r][lane]);
    release(P.fin + tc.x, lane);
    return true;
}

// WB(P): every TRSM chunk of P has read its unfactored diagonal block in
// place, so the factored block (scratch, column-major w x w) goes back into
// the values; lane = block row.
__device__ bool task_wb(const SnParams &P, int4 ta, int lane, unsigned long long *tr) {
    const int Pi = ta.y, p0 = ta.z, w = ta.w - ta.z;
    const int4 pm = __ldg(P.panm + Pi);
    int dcl, clol;
    panel_cols(P, p0, w, lane, dcl, clol);
    if (!wait_ge(P, P.cnt + 2 * Pi + 1, (unsigned)pm.y, lane)) return false;
    if (tr && lane == 0) tr[1] = tr[2] = globaltimer();
    for (int c = 0; c < w; c++) {
        const int dc = __shfl_sync(0xffffffffu, dcl, c), clo = __shfl_sync(0xffffffffu, clol, c);
        if (lane < w && lane >= clo) stv(P.v + dc + (lane - c), ldv(P.dblk + pm.z + c * w + lane));
    }
    release(P.fin + Pi, lane);
    return true;
}

// RG: consecutive pushes from one-column source panels into K (at most
// kRgPushes, each at most kRgRows / 4 rows below its column), applied in
// order by this warp on a shared-memory image of the slots they touch.  A
// one-column panel is a one-column supernode: its rows below all sit in
// R_S.  Lane i holds push i's records.  Before the target wait the warp
// stages the MAC indices (u16; pair q, row t of push i at its offset +
// q * h + t) and the multiplier indices; after it, the slot values.  The
// source panels' TRSM counters are acquired lane-parallel; the pushes whose
// sources are factored get their L rows loaded together, then run back to
// back from shared memory (a warp barrier between pushes), so the chain
// into K costs ~0.1 us per push.  The slots are stored back and every push's
// RECT chunks counted at the end.
__device__ bool task_rg(const SnParams &P, RgSmem &G, int4 ta, int4 tb, int4 tc, int lane,
                        unsigned long long *tr) {
    const int idx0 = ta.y, uidx0 = ta.z, nchunks = ta.w;
    const int slot0 = tb.x, nslot = tb.y, x0 = tb.z, m = tb.w;
    int4 ps = make_int4(0, 0, 0, 0), pn = make_int4(0, 1, 0, 0);
    int dcl = 0, fneed = 0;
    if (lane < m) {
        ps = __ldg(P.push + x0 + lane);
        pn = __ldg(P.pan + ps.x);
        dcl = __ldg(P.diag_pos + pn.x);
        fneed = __ldg(&P.panm[ps.x].y);
    }
    // per push: offsets of its MAC indices, multiplier indices and L rows
    // (exclusive scans over the lanes)
    const int npl = ps.z - ps.y, nmac = npl * pn.w;
    int ioff = nmac, uoff = npl, loff = lane < m ? pn.w : 0;
    const int hl = loff;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int a = __shfl_up_sync(0xffffffffu, ioff, d), b = __shfl_up_sync(0xffffffffu, uoff, d),
                  c = __shfl_up_sync(0xffffffffu, loff, d);
        if (lane >= d) {
            ioff += a;
            uoff += b;
            loff += c;
        }
    }
    ioff -= nmac;
    uoff -= npl;
    loff -= hl;
    const int nidx = __shfl_sync(0xffffffffu, ioff + nmac, 31), nuidx = __shfl_sync(0xffffffffu, uoff + npl, 31);
    for (int e = lane; e < nidx; e += 32) G.idx[e] = __ldg(P.rg_idx + idx0 + e);
    for (int e = lane; e < nuidx; e += 32) G.uidx[e] = __ldg(P.rg_uidx + uidx0 + e);
    int slot[kRgSlots / 32];
#pragma unroll
    for (int j = 0; j < kRgSlots / 32; j++) slot[j] = lane + 32 * j < nslot ? __ldg(P.rg_slot + slot0 + lane + 32 * j) : -1;
    // Stage the L rows of the pushes whose sources are factored (lane i
    // acquires push i's TRSM counter): [staged, e) -> flat rows of G.L,
    // asynchronously.  Returns false on the error path.
    int staged = 0;
    const unsigned long long t0 = globaltimer();
    auto stage = [&](bool block) -> bool {
        while (true) {
            const bool rdy = lane < staged || lane >= m || ld_acquire(P.cnt + 2 * ps.x + 1) >= (unsigned)fneed;
            const unsigned nr = __ballot_sync(0xffffffffu, rdy) | (m < 32 ? ~0u << m : 0u);
            const int e = nr == ~0u ? m : min(m, __ffs(~nr) - 1);
            if (e > staged) {
                __syncwarp();
                const int r0 = __shfl_sync(0xffffffffu, loff, staged);
                const int r1 = __shfl_sync(0xffffffffu, loff + hl, e - 1);
                const int nit = (r1 - r0 + 31) >> 5;  // the same trip count on every lane (shuffles inside)
#pragma unroll 1
                for (int it = 0; it < nit; it++) {
                    const int r = r0 + lane + 32 * it;
                    // the push holding flat row r: the last push k < e with loff(k) <= r
                    int k = staged;
#pragma unroll
                    for (int step = kRgPushes / 2; step; step >>= 1) {
                        const int c = k + step;
                        const int lc = __shfl_sync(0xffffffffu, loff, c & 31);
                        if (c < e && lc <= r) k = c;
                    }
                    const int lk = __shfl_sync(0xffffffffu, loff, k), dk = __shfl_sync(0xffffffffu, dcl, k);
                    if (r < r1) cp_async8(&G.L[r], P.v + dk + 1 + (r - lk), true, P.v);
                }
                staged = e;
                return true;
            }
            if (!block) return true;
            if (*(volatile int *)P.err) return false;
            if (globaltimer() - t0 > kSnWatchdogNs) {
                if (lane == 0) atomicExch(P.err, 1);
                return false;
            }
            __nanosleep(64);
        }
    };
    // lane 31 (no push) polls the target alongside the first staging round
    unsigned tv = 0;
    if (lane == 31) tv = ld_acquire(P.cnt + 2 * tc.x);
    stage(false);  // sources are usually factored long before the target is ready
    __syncwarp();
    const bool tgt_ok = __shfl_sync(0xffffffffu, (int)(tv >= (unsigned)tc.y), 31) != 0;
    if (!tgt_ok && !wait_ge(P, P.cnt + 2 * tc.x, (unsigned)tc.y, lane)) return false;
    if (tr && lane == 0) tr[1] = tr[2] = globaltimer();
#pragma unroll
    for (int j = 0; j < kRgSlots / 32; j++)
        if (slot[j] >= 0) G.val[lane + 32 * j] = ldv(P.v + slot[j]);
    int done = 0;
    while (done < m) {
        if (staged == done && !stage(true)) return false;
        cp_async_wait();
        __syncwarp();
        for (int k = done; k < staged; k++) {
            const int h = __shfl_sync(0xffffffffu, pn.w, k), np_ = __shfl_sync(0xffffffffu, npl, k);
            const int io = __shfl_sync(0xffffffffu, ioff, k), uo = __shfl_sync(0xffffffffu, uoff, k);
            const int lo = __shfl_sync(0xffffffffu, loff, k);
            for (int t = lane; t < h; t += 32) {
                const double L = G.L[lo + t];
                for (int q = 0; q < np_; q++) {
                    const double u = G.val[G.uidx[uo + q]];
                    const int ix = G.idx[io + q * h + t];
                    G.val[ix] = msub(G.val[ix], L, u);
                }
            }
            __syncwarp();  // the next push sees these updates
        }
        done = staged;
        if (done < m) stage(false);
    }
#pragma unroll
    for (int j = 0; j < kRgSlots / 32; j++)
        if (slot[j] >= 0) stv(P.v + slot[j], G.val[lane + 32 * j]);
    __syncwarp();
    if (lane == 0) {
        __threadfence();
        atomicAdd(P.cnt + 2 * tc.x, (unsigned)nchunks);
    }
    return true;
}

__device__ __forceinline__ bool run_task(const SnParams &P, WarpSmem &S, int4 ta, int4 tb, int4 tc, int lane,
                                         unsigned long long *tr) {
    const int kind = (int)((unsigned)ta.x >> 29);  // code = kind << 2 | flags in bits 27-31
    if (kind == kSnRg) return task_rg(P, S.g, ta, tb, tc, lane, tr);
    const int w = ta.w - ta.z;
    if (kind == kSnTrsm) {
        const int4 pm = __ldg(P.panm + ta.y);
        if (!wait_ge(P, P.cnt + 2 * ta.y, (unsigned)pm.x, lane)) return false;
        if (tr && lane == 0) tr[1] = tr[2] = globaltimer();
        if (w == 1) task_trsm1(P, ta, tb, lane);
        else task_trsm(P, S.t, ta, tb, pm, lane, tr);
        release(P.cnt + 2 * ta.y + 1, lane);
        return true;
    }
    if (kind == kSnUw) return task_uw(P, S.r, ta, tb, tc, lane, tr);
    if (kind == kSnWb) return task_wb(P, ta, lane, tr);
    const bool ok = w == 1 ? task_rect1(P, ta, tb, tc, lane, tr) : task_rect(P, S.r, ta, tb, tc, lane, tr);
    if (ok) release(P.cnt + 2 * tc.x, lane);
    return ok;
}

// Task assignment: each warp walks its own list, [wptr[g], wptr[g + 1]) of
// the warp-major task array (built at upload, sn_assign).  A warp's tasks
// keep their list order and every dependency has a smaller list index
// (record tc.w), so the smallest unfinished task can always run: no deadlock.
__global__ void __launch_bounds__(kSnThreads, 2) sn_kernel(SnParams P) {
    extern __shared__ __align__(16) unsigned char sn_smem_raw[];
    WarpSmem *smem = reinterpret_cast<WarpSmem *>(sn_smem_raw);
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    WarpSmem &S = smem[wib];
    const int g = blockIdx.x * kSnWarps + wib;
    int pos = __ldg(P.wptr + g);
    const int end = __ldg(P.wptr + g + 1);
    int4 ta = make_int4(0, 0, 0, 0), tb = ta, tc = ta;
    if (pos < end) {
        ta = __ldg(P.tasks + 3 * (size_t)pos);
        tb = __ldg(P.tasks + 3 * (size_t)pos + 1);
        tc = __ldg(P.tasks + 3 * (size_t)pos + 2);
    }
    while (pos < end) {
        // the next task's records load while this one runs
        int4 na = ta, nb = tb, nc = tc;
        if (pos + 1 < end) {
            na = __ldg(P.tasks + 3 * (size_t)pos + 3);
            nb = __ldg(P.tasks + 3 * (size_t)pos + 4);
            nc = __ldg(P.tasks + 3 * (size_t)pos + 5);
        }
        unsigned long long *tr = P.trace ? P.trace + kTraceWords * (size_t)tc.w : nullptr;
        if (tr && lane == 0) {
            tr[0] = globaltimer();
            tr[4] = g;
        }
        if (!run_task(P, S, ta, tb, tc, lane, tr)) return;
        if (tr && lane == 0) tr[3] = globaltimer();
        pos++;
        ta = na;
        tb = nb;
        tc = nc;
    }
}


// pivot test of every column (_kernels.py:60-65): |piv| <= thresh * cmax.
// One warp per column adds the maximum over its final U part and diagonal
// (rows <= c, never divided) to the undivided-L maxima the tasks gathered.
__global__ void sn_check_kernel(const double *v, const i32 *col_ptr, const i32 *diag_pos,
                                const unsigned long long *cmax, const i32 *fail_level, i32 n,
                                double thresh, int by_column, unsigned long long *fail) {
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    for (i32 c = gw; c < n; c += nw) {
        const int d = __ldg(diag_pos + c);
        unsigned long long m = 0;
        for (int q = __ldg(col_ptr + c) + lane; q <= d; q += 32) {
            const unsigned long long b = absbits(__ldcg(v + q));
            m = b > m ? b : m;
        }
        m = warp_max(m);
        if (lane == 0) {
            const unsigned long long l = cmax[c];
            m = l > m ? l : m;
            const double piv = __ldcg(v + d);
            if (fabs(piv) <= __dmul_rn(thresh, __longlong_as_double((long long)m))) {
                const unsigned long long key =
                    by_column ? (unsigned long long)c
                              : (((unsigned long long)__ldg(fail_level + c)) << 32) | (unsigned)c;
                atomicMin(fail, key);
            }
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

// Warp assignment.  Default: round-robin over the list (task i -> CTA
// i % grid, warp (i / grid) % 8, consecutive tasks on different SMs).
// GLU_SN_ASSIGN=sim: a list-scheduling simulation of the kernel under the
// plan's latency model -- tasks in list order, each on the warp that frees
// first, starting when its counters would be met -- measured slightly
// slower (cfg4 52.1 vs 50.5 ms, g400 8.03 vs 7.65 ms; assigning each task to
// the least-loaded warp: 52.8 / 8.33 ms): round-robin also spreads
// consecutive, mostly independent tasks over different SMs.  Returns the warp-major
// records (tc.w = list index) and per-warp ranges.
static void sn_assign(const SnPlan *p, int W, std::vector<int4> &tw, std::vector<int> &wptr) {
    constexpr double kHop = 2.5;
    const i64 n = (i64)p->tasks.size() / 3, np = (i64)p->pan.size();
    std::vector<double> fdone(np, 0.0), kprev(np, 0.0), kcur(np, 0.0);
    std::vector<i32> kowner(np, -1);  // push (or -1 - RG) whose tasks kcur collects
    std::vector<i32> warp(n);
    using E = std::pair<double, int>;
    std::priority_queue<E, std::vector<E>, std::greater<E>> freeq;
    for (int w = 0; w < W; w++) freeq.push({0.0, w});
    const char *mode = std::getenv("GLU_SN_ASSIGN");
    const bool sim = mode && std::string(mode) == "sim";
    const int grid = W / kSnWarps;
    auto settle = [&](i64 K, i32 owner) {  // a new push (group) into K: earlier ones are complete
        if (kowner[K] != owner) {
            kprev[K] = std::max(kprev[K], kcur[K]);
            kcur[K] = 0.0;
            kowner[K] = owner;
        }
    };
    for (i64 i = 0; i < n && !sim; i++) warp[i] = (int)((i % grid) * kSnWarps + (i / grid) % kSnWarps);
    for (i64 i = 0; i < n && sim; i++) {
        const I4 a = p->tasks[3 * i], b = p->tasks[3 * i + 1], c = p->tasks[3 * i + 2];
        const int kind = (a.x >> 27) >> 2;
        double ready = 0.0;
        if (kind == kSnTrsm) {
            const i64 Pn = a.y;
            settle(Pn, -2);
            ready = kprev[Pn];
        } else if (kind == kSnRect) {
            const i64 K = c.x;
            // chunks of one push share (need); a different need means a new push
            settle(K, c.y);
            ready = std::max(fdone[a.y], kprev[K]);
        } else if (kind == kSnWb) {
            ready = fdone[a.y];
        } else if (kind == kSnUw) {
            const i64 K = c.x;
            ready = kowner[K] == c.y ? std::max(kprev[K], kcur[K]) : kprev[K];
        } else {  // RG: the target once, then every source as it goes
            const i64 K = c.x;
            settle(K, c.y);
            ready = kprev[K];
            for (i64 y = b.z; y < b.z + b.w; y++) ready = std::max(ready, fdone[p->push[y].x]);
        }
        ready += kHop;
        const E f = freeq.top();
        freeq.pop();
        const double fin = std::max(ready, f.first) + (double)p->task_cost[i];
        freeq.push({fin, f.second});
        warp[i] = f.second;
        if (kind == kSnTrsm) fdone[a.y] = std::max(fdone[a.y], fin);
        else if (kind == kSnRect || kind == kSnRg) kcur[c.x] = std::max(kcur[c.x], fin);
    }
    wptr.assign(W + 1, 0);
    for (i64 i = 0; i < n; i++) wptr[warp[i] + 1]++;
    for (int w = 0; w < W; w++) wptr[w + 1] += wptr[w];
    std::vector<int> at(wptr.begin(), wptr.end() - 1);
    tw.resize(3 * n);
    for (i64 i = 0; i < n; i++) {
        const i64 q = at[warp[i]]++;
        for (int r = 0; r < 3; r++) {
            const I4 t = p->tasks[3 * i + r];
            tw[3 * q + r] = make_int4(t.x, t.y, t.z, r == 2 ? (int)i : t.w);
        }
    }
}

struct SnDev {
    int4 *pairs = nullptr, *tasks = nullptr, *panm = nullptr, *push = nullptr, *pan = nullptr;
    i32 *relmap = nullptr, *col_a = nullptr, *rg_slot = nullptr;
    uint16_t *rg_idx = nullptr, *rg_uidx = nullptr;
    double *dblk = nullptr;
    i64 n = 0, n_tasks = 0, n_pan = 0;
    unsigned *cnt = nullptr;  // 2 per panel + the ticket counter
    unsigned *fin = nullptr;  // per panel: WB / UW tasks done
    unsigned long long *cmax = nullptr;
    unsigned long long *trace = nullptr;  // per-task timestamps (diagnostics)
    int grid = 0;
    // host copy-out of final panels (sn_copy_out)
    std::vector<int32_t> h_p1, h_nch, h_fin;  // per panel: end column, TRSM chunks, final completions
    std::vector<int64_t> h_colptr;
    unsigned *h_poll = nullptr;               // pinned: a window of counters
    cudaStream_t s_poll = nullptr, s_copy = nullptr;
    cudaEvent_t ev_done = nullptr;
    int *wptr = nullptr;  // per-warp task ranges (sn_assign)
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
    if (d->h_poll) cudaFreeHost(d->h_poll);
    if (d->s_poll) cudaStreamDestroy(d->s_poll);
    if (d->s_copy) cudaStreamDestroy(d->s_copy);
    if (d->ev_done) cudaEventDestroy(d->ev_done);
    void *ptrs[] = {d->pairs, d->tasks, d->panm,  d->push,   d->pan,     d->relmap, d->col_a,
                    d->dblk,  d->cnt,   d->cmax,  d->trace, d->rg_slot, d->rg_idx, d->rg_uidx, d->wptr, d->fin};
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
    if (e == cudaSuccess) e = up(&d->pairs, cast(p->pairs), bytes);

    if (e == cudaSuccess) e = up(&d->panm, cast(p->panm), bytes);
    if (e == cudaSuccess) e = up(&d->push, cast(p->push), bytes);
    if (e == cudaSuccess) e = up(&d->pan, cast(p->pan), bytes);
    if (e == cudaSuccess) e = up(&d->rg_slot, p->rg_slot, bytes);
    if (e == cudaSuccess) e = up(&d->rg_idx, p->rg_idx, bytes);
    if (e == cudaSuccess) e = up(&d->rg_uidx, p->rg_uidx, bytes);
    if (e == cudaSuccess) e = up(&d->relmap, p->relmap, bytes);
    if (e == cudaSuccess) e = up(&d->col_a, p->col_a, bytes);
    d->n = p->n;
    d->n_tasks = (i64)p->tasks.size() / 3;
    d->h_colptr = p->col_ptr_h;
    d->h_p1.resize(p->pan.size());
    d->h_nch.resize(p->pan.size());
    d->h_fin.resize(p->pan.size());
    for (size_t q = 0; q < p->pan.size(); q++) {
        d->h_p1[q] = p->pan[q].y;
        d->h_nch[q] = p->panm[q].y;
        d->h_fin[q] = p->panm[q].w;
    }
    d->n_pan = (i64)p->pan.size();
    if (e == cudaSuccess && p->n_dblk > 0) {
        e = cudaMalloc((void **)&d->dblk, sizeof(double) * p->n_dblk);
        *bytes += (i64)sizeof(double) * p->n_dblk;
    }
    if (e == cudaSuccess) e = cudaMalloc((void **)&d->cnt, sizeof(unsigned) * (2 * d->n_pan + 32));
    if (e == cudaSuccess) e = cudaMalloc((void **)&d->fin, sizeof(unsigned) * std::max<i64>(d->n_pan, 1));
    if (e == cudaSuccess) e = cudaMalloc((void **)&d->cmax, sizeof(unsigned long long) * std::max<i64>(d->n, 1));
    if (e != cudaSuccess) {
        set_error(std::string("supernodal plan upload: ") + cudaGetErrorString(e));
        sn_free(d);
        return GLU_ECUDA;
    }
    *bytes += (i64)(sizeof(unsigned) * 2 * d->n_pan + sizeof(unsigned long long) * d->n);
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    d->grid = sn_grid(sms);
    if (d->grid <= 0) {
        set_error("supernodal kernel cannot be co-resident");
        sn_free(d);
        return GLU_ECUDA;
    }
    {  // tasks in warp-major order (sn_assign), each record carrying its list index
        std::vector<int4> tw;
        std::vector<int> wptr;
        sn_assign(p, d->grid * kSnWarps, tw, wptr);
        e = up(&d->tasks, tw, bytes);
        if (e == cudaSuccess) e = up(&d->wptr, wptr, bytes);
        if (e != cudaSuccess) {
            set_error(std::string("supernodal plan upload: ") + cudaGetErrorString(e));
            sn_free(d);
            return GLU_ECUDA;
        }
    }
    *out = d;
    return GLU_OK;
}

int64_t sn_set_trace(SnDev *d, int mode) {
    // 1: per-task trace, 0: off
    if (mode && !d->trace) {
        if (cudaMalloc((void **)&d->trace, sizeof(unsigned long long) * kTraceWords * std::max<i64>(d->n_tasks, 1)) !=
            cudaSuccess) {
            set_error("cudaMalloc(task trace)");
            return GLU_ECUDA;
        }
    } else if (!mode && d->trace) {
        cudaFree(d->trace);
        d->trace = nullptr;
    }
    return GLU_OK;
}

int64_t sn_read_trace(SnDev *d, int64_t *out, int64_t max_tasks) {
    if (!d->trace) return 0;
    const i64 m = std::min<i64>(max_tasks, d->n_tasks);
    if (cudaMemcpy(out, d->trace, sizeof(unsigned long long) * kTraceWords * m, cudaMemcpyDeviceToHost) != cudaSuccess)
        return GLU_ECUDA;
    return m;
}

int64_t sn_copy_out(SnDev *d, const double *v, double *out, void *stream) {
    constexpr i64 kWin = 1 << 18;            // panels polled per round trip
    constexpr i64 kMinRun = 1ll << 17;       // smallest early copy (doubles: 1 MB)
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = cudaSuccess;
    if (!d->h_poll) {
        e = cudaHostAlloc((void **)&d->h_poll, sizeof(unsigned) * 3 * kWin, cudaHostAllocDefault);
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&d->s_poll, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&d->s_copy, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&d->ev_done, cudaEventDisableTiming);
        if (e != cudaSuccess) {
            set_error(std::string("sn_copy_out: ") + cudaGetErrorString(e));
            return GLU_ECUDA;
        }
    }
    const i64 np = d->n_pan;
    if ((e = cudaEventRecord(d->ev_done, s)) != cudaSuccess) {
        set_error(std::string("sn_copy_out: ") + cudaGetErrorString(e));
        return GLU_ECUDA;
    }
    // A panel is final once every TRSM chunk, and the WB / UW tasks writing
    // its columns, have counted themselves.  While the kernel runs, windows
    // of the counters are polled (a cursor sweeping the panels not yet
    // copied) and every run of final, not yet copied panels worth >= 1 MB is
    // copied out; in nested-dissection order whole subtrees finish while
    // their ancestors' separators are still being factored.
    std::vector<char> copied((size_t)np, 0);
    auto slots = [&](i64 p) { return d->h_colptr[p > 0 ? d->h_p1[p - 1] : 0]; };  // first slot of panel p
    auto copy_run = [&](i64 a, i64 b) {  // panels [a, b)
        const i64 s0 = slots(a), s1 = d->h_colptr[d->h_p1[b - 1]];
        std::fill(copied.begin() + a, copied.begin() + b, (char)1);
        return cudaMemcpyAsync(out + s0, v + s0, sizeof(double) * (s1 - s0), cudaMemcpyDeviceToHost, d->s_copy);
    };
    i64 lo = 0, cur = 0;
    unsigned *hc = d->h_poll, *hf = d->h_poll + 2 * kWin;
    while (lo < np && cudaEventQuery(d->ev_done) == cudaErrorNotReady) {
        if (cur >= np) cur = lo;
        const i64 len = std::min<i64>(kWin, np - cur);
        e = cudaMemcpyAsync(hc, d->cnt + 2 * cur, sizeof(unsigned) * 2 * len, cudaMemcpyDeviceToHost, d->s_poll);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(hf, d->fin + cur, sizeof(unsigned) * len, cudaMemcpyDeviceToHost, d->s_poll);
        if (e == cudaSuccess) e = cudaStreamSynchronize(d->s_poll);
        if (e != cudaSuccess) break;
        bool issued = false;
        for (i64 q = 0; q < len && e == cudaSuccess;) {
            const i64 p = cur + q;
            auto fin = [&](i64 r) {
                return hc[2 * r + 1] >= (unsigned)d->h_nch[cur + r] && hf[r] >= (unsigned)d->h_fin[cur + r];
            };
            if (copied[p] || !fin(q)) {
                q++;
                continue;
            }
            i64 r = q;
            while (r < len && !copied[cur + r] && fin(r)) r++;
            // a run reaching the copied prefix or worth >= 1 MB goes now
            if (p == lo || slots(cur + r) - slots(p) >= kMinRun) {
                e = copy_run(p, cur + r);
                issued = true;
            }
            q = r;
        }
        while (lo < np && copied[lo]) lo++;
        cur += len;
        if (!issued) std::this_thread::sleep_for(std::chrono::microseconds(100));
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    for (i64 p = lo; p < np && e == cudaSuccess;) {  // the rest, in maximal runs
        if (copied[p]) {
            p++;
            continue;
        }
        i64 r = p;
        while (r < np && !copied[r]) r++;
        e = copy_run(p, r);
        p = r;
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(d->s_copy);
    if (e != cudaSuccess) {
        set_error(std::string("sn_copy_out: ") + cudaGetErrorString(e));
        return GLU_ECUDA;
    }
    return GLU_OK;
}

int64_t sn_launch(SnDev *d, double *v, const int32_t *col_ptr, const int32_t *diag_pos,
                  const int32_t *fail_level, int32_t n, double thresh, bool by_column,
                  unsigned long long *fail, int *err, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(d->cnt, 0, sizeof(unsigned) * (2 * d->n_pan + 32), s);
    if (e == cudaSuccess) e = cudaMemsetAsync(d->fin, 0, sizeof(unsigned) * std::max<i64>(d->n_pan, 1), s);
    if (e == cudaSuccess) e = cudaMemsetAsync(d->cmax, 0, sizeof(unsigned long long) * std::max<i64>(d->n, 1), s);
    if (d->trace && e == cudaSuccess)
        e = cudaMemsetAsync(d->trace, 0, sizeof(unsigned long long) * kTraceWords * std::max<i64>(d->n_tasks, 1), s);
    if (e != cudaSuccess) {
        set_error(std::string("sn_launch: ") + cudaGetErrorString(e));
        return GLU_ECUDA;
    }
    if (d->n_tasks > 0) {
        SnParams P;
        P.v = v;
        P.dblk = d->dblk;
        P.diag_pos = diag_pos;
        P.col_a = d->col_a;
        P.pairs = d->pairs;
        P.tasks = d->tasks;
        P.panm = d->panm;
        P.push = d->push;
        P.pan = d->pan;
        P.rg_slot = d->rg_slot;
        P.rg_idx = d->rg_idx;
        P.rg_uidx = d->rg_uidx;
        P.relmap = d->relmap;
        P.n_tasks = (i32)d->n_tasks;
        P.cnt = d->cnt;
        P.fin = d->fin;
        P.cmax = d->cmax;
        P.err = err;
        P.trace = d->trace;
        P.wptr = d->wptr;
        void *args[] = {&P};
        e = cudaLaunchCooperativeKernel((const void *)sn_kernel, dim3(d->grid), dim3(kSnThreads), args, kSnSmem, s);
        if (e != cudaSuccess) {
            set_error(std::string("sn_kernel: ") + cudaGetErrorString(e));
            return GLU_ECUDA;
        }
    }
    if (n > 0) {
        sn_check_kernel<<<std::min<i64>((n + 7) / 8, 4736), 256, 0, s>>>(v, col_ptr, diag_pos, d->cmax, fail_level,
                                                                        n, thresh, by_column ? 1 : 0, fail);
        e = cudaGetLastError();
        if (e != cudaSuccess) {
            set_error(std::string("sn_check_kernel: ") + cudaGetErrorString(e));
            return GLU_ECUDA;
        }
    }
    return GLU_OK;
}

}  // namespace glu
