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
constexpr int kDoneStride = 8;  // u32 words between phase counters
constexpr int kGdoneRep = 8;    // replicas of the phases-complete counter (spread the pollers)
constexpr int kLine = 32;       // u32 words per 128-byte line
constexpr unsigned long long kSnWatchdogNs = 4000000000ull;

struct SnParams {
    double *v;
    const i32 *col_ptr, *diag_pos, *col_a, *fail_level;
    const int4 *pairs, *tasks;  // tasks: 2 records each (glu_internal.h SnPlan::tasks)
    const i32 *relmap, *phase_ptr;
    i32 n_tasks;
    unsigned *done;   // per phase: counted tasks (kDoneStride apart)
    unsigned *gdone;  // phases complete, kGdoneRep replicas kLine apart
    unsigned long long *cmax;
    int *err;
    unsigned long long *stamps;  // optional: [0] kernel start, [1 + p] completion of phase p
    unsigned long long *trace;   // optional: per task {iteration start, wait done, executed, 0}
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

constexpr int kB = 32;  // lanes: shared-memory block dimension
struct WarpSmem {
    double b[kB][kB + 1];  // panel block, column-major [column][row]
    int clo[kB];           // per panel column: first panel row present
    double pad[16 * kB - kB + 8];  // RectSmem (task_rect_tile) overlays this region
};

// Compile-time loop: f(std::integral_constant<int, I>) for I in [B, E).  The
// FP64 chains below index register arrays with the loop counter, which
// must be a constant after unrolling (a nest of #pragma unroll loops whose
// body holds the division's slow-path call is left rolled by nvcc, and the
// arrays then live in local memory).
template <int B, int E, class F>
__device__ __forceinline__ void static_for(F &&f) {
    if constexpr (B < E) {
        f(std::integral_constant<int, B>{});
        static_for<B + 1, E>(f);
    }
}

// Panel metadata, lane = panel column: its diagonal slot and the first
// panel row present in it (a supernode's U rows in a column are a suffix).
// Loaded lane-parallel so the block loads below issue back to back.
__device__ __forceinline__ void panel_cols(const SnParams &P, int p0, int w, int lane, int &dc, int &clo) {
    dc = 0;
    clo = kB;
    if (lane < w) {
        dc = __ldg(P.diag_pos + p0 + lane);
        clo = max(__ldg(P.col_a + p0 + lane) - p0, 0);
    }
}

// The unrolled task variants below run every loop to the class width WM
// without per-width branches: registers of columns / rows >= w hold
// garbage that is never stored (and never feeds a stored value -- a column
// only receives updates from lower columns), so the FP64 chains are free
// of branches and the compiler can interleave them.  Structural
// predicates that change stored values (a supernode's partial U suffix,
// col_a) become selects, never a subtraction of a zero product: x - l * 0
// is not always x (x = -0 with l < 0, or l = inf).

// DIAG: the w x w block of the panel, lane = block row r holding its row
// in registers.  Step j: row j is final for columns >= j (U part), lane j
// broadcasts it; every lane r > j takes column j's undivided value (the
// column maximum over the block's L part -- the U rows are taken by the
// check pass), divides it by the pivot and updates its later columns, so
// every element receives its sources j in ascending order.
template <int WM>
__device__ __forceinline__ void diag_factor(const SnParams &P, int p0, int w, int lane, int dcl, int clol,
                                            double (&x)[WM], unsigned long long &mymax) {
#pragma unroll
    for (int c = 0; c < WM; c++) {
        const int dc = __shfl_sync(0xffffffffu, dcl, c), clo = __shfl_sync(0xffffffffu, clol, c);
        x[c] = (c < w && lane < w && lane >= clo) ? ldv(P.v + dc + (lane - c)) : 0.0;
    }
    mymax = 0;
    static_for<0, WM>([&](auto jc) {
        constexpr int j = decltype(jc)::value;
        const bool below = lane > j && lane < w;
        // bit c: U(j, c) present (column c's U suffix starts at or above row j)
        const unsigned has = __ballot_sync(0xffffffffu, clol <= j);
        const unsigned long long m = warp_max(below ? absbits(x[j]) : 0ull);
        if (lane == j) mymax = m;
        const double piv = __shfl_sync(0xffffffffu, x[j], j);
        const double l = __ddiv_rn(x[j], piv);
        x[j] = below ? l : x[j];
#pragma unroll
        for (int c = j + 1; c < WM; c++) {
            const double ujc = __shfl_sync(0xffffffffu, x[c], j);
            const double y = msub(x[c], l, ujc);
            x[c] = (below && ((has >> c) & 1u)) ? y : x[c];
        }
    });
}

template <int WM>
__device__ void task_diag(const SnParams &P, int4 ta, int lane) {
    const int p0 = ta.z, w = ta.w - ta.z;
    int dcl, clol;
    panel_cols(P, p0, w, lane, dcl, clol);
    double x[WM];
    unsigned long long mymax;
    diag_factor<WM>(P, p0, w, lane, dcl, clol, x, mymax);
#pragma unroll
    for (int c = 0; c < WM; c++) {
        const int dc = __shfl_sync(0xffffffffu, dcl, c), clo = __shfl_sync(0xffffffffu, clol, c);
        if (c < w && lane < w && lane >= clo) stv(P.v + dc + (lane - c), x[c]);
    }
    if (lane < w && mymax) atomicMax(P.cmax + p0 + lane, mymax);
}

// TRSM: 32 rows below the panel; lane = row, the row's w values in
// registers; step j takes the undivided value's maximum, divides, and
// updates the later columns with U(j, c) from the factored block (shared
// memory, broadcast reads).
template <int WM>
__device__ void task_trsm(const SnParams &P, WarpSmem &S, int4 ta, int4 tb, int lane, bool local) {
    const int chunk = ta.x & 0x07ffffff;
    const int p0 = ta.z, p1 = ta.w, w = p1 - p0, h = tb.y;
    int dcl, clol;
    panel_cols(P, p0, w, lane, dcl, clol);
    const int t = chunk * 32 + lane;
    const bool act = t < h;
    if (local) {  // the panel's own stage: its diagonal block is factored here
        double b[WM];
        unsigned long long unused;
        diag_factor<WM>(P, p0, w, lane, dcl, clol, b, unused);
#pragma unroll
        for (int c = 0; c < WM; c++) S.b[c][lane] = lane <= c ? b[c] : 0.0;
    } else {
#pragma unroll
        for (int c = 0; c < WM; c++) {
            const int dc = __shfl_sync(0xffffffffu, dcl, c), clo = __shfl_sync(0xffffffffu, clol, c);
            S.b[c][lane] = (c < w && lane <= c && lane >= clo) ? ldv(P.v + dc + (lane - c)) : 0.0;
        }
    }
    double x[WM];
#pragma unroll
    for (int c = 0; c < WM; c++) {
        const int dc = __shfl_sync(0xffffffffu, dcl, c);
        x[c] = (act && c < w) ? ldv(P.v + dc + (p1 - p0 - c) + t) : 0.0;
    }
    __syncwarp();
    unsigned long long mymax = 0;
    static_for<0, WM>([&](auto jc) {
        constexpr int j = decltype(jc)::value;
        const unsigned has = __ballot_sync(0xffffffffu, clol <= j);
        const unsigned long long m = warp_max(act && j < w ? absbits(x[j]) : 0ull);
        if (lane == j) mymax = m;
        const double d = __ddiv_rn(x[j], S.b[j][j]);
        x[j] = d;
#pragma unroll
        for (int c = j + 1; c < WM; c++) {
            const double y = msub(x[c], d, S.b[c][j]);
            x[c] = ((has >> c) & 1u) ? y : x[c];
        }
    });
#pragma unroll
    for (int c = 0; c < WM; c++) {
        const int dc = __shfl_sync(0xffffffffu, dcl, c);
        if (act && c < w) stv(P.v + dc + (p1 - p0 - c) + t, x[c]);
    }
    if (lane < w && mymax) atomicMax(P.cmax + p0 + lane, mymax);
    __syncwarp();
}

// TRI: U(P, k) for every target column k of the push (lane = column):
// forward substitution with the panel's unit-lower block, j ascending.
template <int WM>
__device__ void task_tri(const SnParams &P, WarpSmem &S, int4 ta, int4 tb, int lane, bool local) {
    const int p0 = ta.z, p1 = ta.w, w = p1 - p0, s1 = tb.x;
    int dcl, clol;
    panel_cols(P, p0, w, lane, dcl, clol);
    const int q = tb.z + lane;
    int4 pr = make_int4(0, p1, 0, -1);
    if (q < tb.w) pr = __ldg(P.pairs + q);
    const bool act = pr.y < p1;
    const int lo = max(pr.y - p0, 0);
    if (local) {  // the panel's own stage: its unit-lower block is factored here
        double b[WM];
        unsigned long long unused;
        diag_factor<WM>(P, p0, w, lane, dcl, clol, b, unused);
        // lane r holds row r: L(r, j) = b[j] for r > j; S.b[j][r] = L(r, j)
#pragma unroll
        for (int j = 0; j < WM; j++) S.b[j][lane] = lane > j ? b[j] : 0.0;
    } else {
#pragma unroll
        for (int j = 0; j < WM; j++) {
            const int dj = __shfl_sync(0xffffffffu, dcl, j);
            S.b[j][lane] = (j < w && lane > j && lane < w) ? ldv(P.v + dj + (lane - j)) : 0.0;
        }
    }
    double u[WM];
#pragma unroll
    for (int j = 0; j < WM; j++) u[j] = (act && j < w && j >= lo) ? ldv(P.v + pr.z - (s1 - (p0 + j))) : 0.0;
    __syncwarp();
    static_for<0, WM>([&](auto jc) {
        constexpr int j = decltype(jc)::value;
        const double uj = u[j];
        const bool on = j >= lo;
#pragma unroll
        for (int r = j + 1; r < WM; r++) {
            const double y = msub(u[r], S.b[j][r], uj);
            u[r] = on ? y : u[r];
        }
    });
    if (act) {
#pragma unroll
        for (int r = 0; r < WM; r++)
            if (r < w && r > lo) stv(P.v + pr.z - (s1 - (p0 + r)), u[r]);
    }
    __syncwarp();
}

// RECT for narrow panels (WM <= 8): lane = row, its divided L row in
// registers; target columns in batches of kRectB (their U(j, k), target
// slots and values loaded together, kRectB independent chains per lane),
// U(j, k) broadcast by shuffle, each chain over j ascending.
constexpr int kRectB = 4;

template <int WM>
__device__ void task_rect(const SnParams &P, int4 ta, int4 tb, int lane) {
    const int chunk = ta.x & 0x07ffffff;
    const int p0 = ta.z, p1 = ta.w, w = p1 - p0, h = tb.y;
    const int s1 = tb.x, in_sn = s1 - p1;
    const int t = chunk * 32 + lane;
    const bool act = t < h;
    const int npair = tb.w - tb.z;
    int4 myp = make_int4(0, p1, 0, -1);
    if (lane < npair) myp = __ldg(P.pairs + tb.z + lane);
    const int dcl = lane < w ? __ldg(P.diag_pos + p0 + lane) : 0;
    double L[WM];
#pragma unroll
    for (int j = 0; j < WM; j++) {
        const int dj = __shfl_sync(0xffffffffu, dcl, j);
        L[j] = (act && j < w) ? ldv(P.v + dj + (p1 - p0 - j) + t) : 0.0;
    }
    for (int q0 = 0; q0 < npair; q0 += kRectB) {
        double uv[kRectB], x[kRectB];
        int pos[kRectB], lo[kRectB];
#pragma unroll
        for (int b = 0; b < kRectB; b++) {
            const int q = q0 + b;
            const int a = __shfl_sync(0xffffffffu, myp.y, q & 31);
            const int base = __shfl_sync(0xffffffffu, myp.z, q & 31);
            const int map = __shfl_sync(0xffffffffu, myp.w, q & 31);
            const bool ok = q < npair && a < p1;
            lo[b] = ok ? max(a - p0, 0) : WM;
            uv[b] = (ok && lane < w && lane >= lo[b]) ? ldv(P.v + base - (s1 - (p0 + lane))) : 0.0;
            pos[b] = -1;
            if (ok && act)
                pos[b] = t < in_sn ? base - (in_sn - t)
                                   : (map >= 0 ? __ldg(P.relmap + map + (t - in_sn)) : base + (t - in_sn));
        }
#pragma unroll
        for (int b = 0; b < kRectB; b++) x[b] = pos[b] >= 0 ? ldv(P.v + pos[b]) : 0.0;
#pragma unroll
        for (int j = 0; j < WM; j++) {
#pragma unroll
            for (int b = 0; b < kRectB; b++) {
                const double uj = __shfl_sync(0xffffffffu, uv[b], j);
                const double y = msub(x[b], L[j], uj);
                x[b] = (j >= lo[b] && j < w) ? y : x[b];
            }
        }
#pragma unroll
        for (int b = 0; b < kRectB; b++)
            if (pos[b] >= 0) stv(P.v + pos[b], x[b]);
    }
}

// RECT for wide panels (w > 8): register-tiled blocks C[32 rows x 16
// target columns] -= L[32 x w] * U[w x 16] (two halves for > 16 target
// columns), every element's chain over j ascending.  Lane (ry, cx) =
// (lane / 4, lane % 4) holds rows ry + 8 i and columns cx + 4 k (i, k < 4);
// per j it reads 4 L and 4 U values from shared memory (conflict-free
// broadcasts) for 16 MACs.  Columns whose U suffix starts inside the panel
// (lo > 0, only in structurally unsymmetric patterns) take the select path.
struct RectSmem {
    double l[kB][kB];  // [j][row]
    double u[kB][16];  // [j][column of the half]
    int lo[16];
};

static_assert(sizeof(RectSmem) <= sizeof(WarpSmem), "RectSmem overlays WarpSmem");

__device__ void task_rect_tile(const SnParams &P, RectSmem &R, int4 ta, int4 tb, int lane) {
    const int chunk = ta.x & 0x07ffffff;
    const int p0 = ta.z, p1 = ta.w, w = p1 - p0, h = tb.y;
    const int s1 = tb.x, in_sn = s1 - p1;
    const int npair = tb.w - tb.z;
    const int t = chunk * 32 + lane;
    int4 myp = make_int4(0, p1, 0, -1);
    if (lane < npair) myp = __ldg(P.pairs + tb.z + lane);
    const bool colok = lane < npair && myp.y < p1;
    const int mylo = colok ? max(myp.y - p0, 0) : kB;
    const int dcl = lane < w ? __ldg(P.diag_pos + p0 + lane) : 0;
#pragma unroll 8
    for (int j = 0; j < kSnW; j++) {
        const int dj = __shfl_sync(0xffffffffu, dcl, j);
        R.l[j][lane] = (t < h && j < w) ? ldv(P.v + dj + (p1 - p0 - j) + t) : 0.0;
    }
    const int ry = lane >> 2, cx = lane & 3;
    for (int half = 0; half * 16 < npair; half++) {
        const int qh = lane - 16 * half;  // this lane's column in the half (lanes 16h .. 16h+15)
        __syncwarp();
        if (qh >= 0 && qh < 16) {
            R.lo[qh] = mylo;
#pragma unroll 8
            for (int j = 0; j < kSnW; j++)
                R.u[j][qh] = (colok && j < w && j >= mylo) ? ldv(P.v + myp.z - (s1 - (p0 + j))) : 0.0;
        }
        const bool anylo = __any_sync(0xffffffffu, qh >= 0 && qh < 16 && colok && mylo > 0);
        double c[4][4];
        int pos[4][4];
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const int q = 16 * half + cx + 4 * k;
            const int base = __shfl_sync(0xffffffffu, myp.z, q & 31), map = __shfl_sync(0xffffffffu, myp.w, q & 31);
            const bool cok = __shfl_sync(0xffffffffu, (int)colok, q & 31) != 0 && q < 32;
#pragma unroll
            for (int i = 0; i < 4; i++) {
                const int tt = chunk * 32 + ry + 8 * i;
                int ps = -1;
                if (cok && tt < h)
                    ps = tt < in_sn ? base - (in_sn - tt)
                                    : (map >= 0 ? __ldg(P.relmap + map + (tt - in_sn)) : base + (tt - in_sn));
                pos[i][k] = ps;
            }
        }
#pragma unroll
        for (int k = 0; k < 4; k++)
#pragma unroll
            for (int i = 0; i < 4; i++) c[i][k] = pos[i][k] >= 0 ? ldv(P.v + pos[i][k]) : 0.0;
        __syncwarp();
        if (!anylo) {
#pragma unroll 4
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
    }
    __syncwarp();
}

// Panel widths in classes 1, 2, 4, 8, 16, 32: every task runs the variant
// unrolled for its class, so the code a phase executes stays small (one
// fully unrolled 32-wide kernel is ~700 KB of SASS, far beyond the
// instruction cache, and most panels are one column wide).
template <int WM>
__device__ __forceinline__ void run_kind(const SnParams &P, WarpSmem &S, int4 ta, int4 tb, int lane) {
    const int code = ta.x >> 27;
    switch (code & ~kSnLocal) {
        case kSnDiag: task_diag<WM>(P, ta, lane); break;
        case kSnTrsm: task_trsm<WM>(P, S, ta, tb, lane, code & kSnLocal); break;
        case kSnTri: task_tri<WM>(P, S, ta, tb, lane, code & kSnLocal); break;
        default:
            if (WM > 8) task_rect_tile(P, *reinterpret_cast<RectSmem *>(&S), ta, tb, lane);
            else task_rect<WM>(P, ta, tb, lane);
            break;
    }
}

__device__ __forceinline__ void run_task(const SnParams &P, WarpSmem &S, int4 ta, int4 tb, int lane) {
    const int w = ta.w - ta.z;
    if (w <= 1) run_kind<1>(P, S, ta, tb, lane);
    else if (w <= 2) run_kind<2>(P, S, ta, tb, lane);
    else if (w <= 4) run_kind<4>(P, S, ta, tb, lane);
    else if (w <= 8) run_kind<8>(P, S, ta, tb, lane);
    else if (kSnW <= 16 || w <= 16) run_kind<16>(P, S, ta, tb, lane);
    else run_kind<(kSnW > 16 ? 32 : 16)>(P, S, ta, tb, lane);
}

// A warp leaving phase p counts its tasks of p (release: fence, then add);
// the warp that completes p advances the phases-complete counter.  Phases
// complete in order (a phase's tasks start after the previous one
// completed), and atomicMax keeps the counter monotone.
__device__ __forceinline__ void flush_phase(const SnParams &P, int p, unsigned mine) {
    __threadfence();
    const unsigned old = atomicAdd(P.done + (size_t)p * kDoneStride, mine);
    if (old + mine == (unsigned)(__ldg(P.phase_ptr + p + 1) - __ldg(P.phase_ptr + p))) {
        if (P.stamps) P.stamps[1 + p] = globaltimer();
#pragma unroll
        for (int r = 0; r < kGdoneRep; r++) atomicMax(P.gdone + r * kLine, (unsigned)(p + 1));
    }
}

struct CtaSync {
    int known;  // phases known complete (from the last poll of this CTA)
    int lock;   // one polling warp per CTA at a time
};

// Wait until phases [0, p) are complete.  Warps of a CTA share one poller:
// the others read the CTA's last observation from shared memory, so an
// SM sends at most one poll at a time to the (replicated) global counter
// instead of one per waiting warp.  False on the watchdog / error path.
__device__ bool wait_phase(const SnParams &P, CtaSync *cs, int p, int lane) {
    bool ok = true;
    if (lane == 0) {
        volatile int *known = &cs->known;
        if (*known < p) {
            const unsigned *g = P.gdone + (blockIdx.x % kGdoneRep) * kLine;
            const unsigned long long t0 = globaltimer();
            while (*known < p) {
                if (atomicCAS(&cs->lock, 0, 1) == 0) {
                    const int seen = (int)ld_acquire(g);
                    atomicMax(&cs->known, seen);
                    atomicExch(&cs->lock, 0);
                    if (seen >= p) break;
                }
                if (*(volatile int *)P.err) { ok = false; break; }
                if (globaltimer() - t0 > kSnWatchdogNs) {
                    atomicExch(P.err, 1);
                    ok = false;
                    break;
                }
                __nanosleep(32);
            }
        }
        __threadfence_block();
    }
    return __shfl_sync(0xffffffffu, (int)ok, 0) != 0;
}

__global__ void __launch_bounds__(kSnThreads, 2) sn_kernel(SnParams P) {
    extern __shared__ __align__(16) unsigned char sn_smem_raw[];
    WarpSmem *smem = reinterpret_cast<WarpSmem *>(sn_smem_raw);
    __shared__ CtaSync cs;
    if (threadIdx.x == 0) {
        cs.known = 0;
        cs.lock = 0;
        if (P.stamps && blockIdx.x == 0) P.stamps[0] = globaltimer();
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    WarpSmem &S = smem[wib];
    const int nw = gridDim.x * kSnWarps;
    int cur = -1;
    unsigned mine = 0;
    int i = wib * gridDim.x + blockIdx.x;
    int4 ta = make_int4(0, 0, 0, 0), tb = ta;
    if (i < P.n_tasks) {
        ta = __ldg(P.tasks + 2 * (size_t)i);
        tb = __ldg(P.tasks + 2 * (size_t)i + 1);
    }
    while (i < P.n_tasks) {
        // the next task's records load while this one runs
        const int inext = i + nw;
        int4 na = ta, nb = tb;
        if (inext < P.n_tasks) {
            na = __ldg(P.tasks + 2 * (size_t)inext);
            nb = __ldg(P.tasks + 2 * (size_t)inext + 1);
        }
        unsigned long long t_start = 0;
        if (P.trace) t_start = globaltimer();
        if (ta.y != cur) {
            if (mine) {
                __syncwarp();
                if (lane == 0) flush_phase(P, cur, mine);
            }
            mine = 0;
            cur = ta.y;
            if (cur > 0 && !wait_phase(P, &cs, cur, lane)) return;
        }
        unsigned long long t_wait = 0;
        if (P.trace) t_wait = globaltimer();
        run_task(P, S, ta, tb, lane);
        if (P.trace && lane == 0) {
            __syncwarp(1u);
            unsigned long long *tr = P.trace + 4 * (size_t)i;
            tr[0] = t_start;
            tr[1] = t_wait;
            tr[2] = globaltimer();
        }
        mine++;
        i = inext;
        ta = na;
        tb = nb;
    }
    if (mine) {
        __syncwarp();
        if (lane == 0) flush_phase(P, cur, mine);
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

struct SnDev {
    int4 *pairs = nullptr, *tasks = nullptr;
    i32 *relmap = nullptr, *phase_ptr = nullptr, *col_a = nullptr;
    i64 n = 0, n_tasks = 0, n_phases = 0;
    unsigned *done = nullptr, *gdone = nullptr;
    unsigned long long *cmax = nullptr;
    unsigned long long *stamps = nullptr;  // per-phase completion times (diagnostics)
    unsigned long long *trace = nullptr;   // per-task timestamps (diagnostics)
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
    void *ptrs[] = {d->pairs, d->tasks, d->relmap, d->phase_ptr, d->col_a, d->done, d->gdone, d->cmax,
                    d->stamps, d->trace};
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
    if (e == cudaSuccess) e = up(&d->tasks, cast(p->tasks), bytes);
    if (e == cudaSuccess) e = up(&d->relmap, p->relmap, bytes);
    if (e == cudaSuccess) e = up(&d->phase_ptr, p->phase_ptr, bytes);
    if (e == cudaSuccess) e = up(&d->col_a, p->col_a, bytes);
    d->n = p->n;
    d->n_tasks = (i64)p->tasks.size() / 2;
    d->n_phases = (i64)p->phase_ptr.size() - 1;
    if (e == cudaSuccess)
        e = cudaMalloc((void **)&d->done, sizeof(unsigned) * kDoneStride * std::max<i64>(d->n_phases, 1));
    if (e == cudaSuccess) e = cudaMalloc((void **)&d->gdone, sizeof(unsigned) * kGdoneRep * kLine);
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

int64_t sn_set_stamps(SnDev *d, int mode) {
    // 1: per-phase stamps, 2: + per-task trace, 0: off
    if (mode && !d->stamps) {
        if (cudaMalloc((void **)&d->stamps, sizeof(unsigned long long) * (d->n_phases + 1)) != cudaSuccess) {
            set_error("cudaMalloc(phase stamps)");
            return GLU_ECUDA;
        }
    } else if (!mode && d->stamps) {
        cudaFree(d->stamps);
        d->stamps = nullptr;
    }
    if (mode == 2 && !d->trace) {
        if (cudaMalloc((void **)&d->trace, sizeof(unsigned long long) * 4 * std::max<i64>(d->n_tasks, 1)) !=
            cudaSuccess) {
            set_error("cudaMalloc(task trace)");
            return GLU_ECUDA;
        }
    } else if (mode != 2 && d->trace) {
        cudaFree(d->trace);
        d->trace = nullptr;
    }
    return GLU_OK;
}

int64_t sn_read_trace(SnDev *d, int64_t *out, int64_t max_tasks) {
    if (!d->trace) return 0;
    const i64 m = std::min<i64>(max_tasks, d->n_tasks);
    if (cudaMemcpy(out, d->trace, sizeof(unsigned long long) * 4 * m, cudaMemcpyDeviceToHost) != cudaSuccess)
        return GLU_ECUDA;
    return m;
}

int64_t sn_read_stamps(SnDev *d, int64_t *out, int64_t max) {
    if (!d->stamps) return 0;
    const i64 m = std::min<i64>(max, d->n_phases + 1);
    std::vector<unsigned long long> h((size_t)m);
    if (cudaMemcpy(h.data(), d->stamps, sizeof(unsigned long long) * m, cudaMemcpyDeviceToHost) != cudaSuccess)
        return GLU_ECUDA;
    for (i64 i = 0; i < m; i++) out[i] = (int64_t)h[i];
    return m;
}

int64_t sn_launch(SnDev *d, double *v, const int32_t *col_ptr, const int32_t *diag_pos,
                  const int32_t *fail_level, int32_t n, double thresh, bool by_column,
                  unsigned long long *fail, int *err, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(d->done, 0, sizeof(unsigned) * kDoneStride * std::max<i64>(d->n_phases, 1), s);
    if (e == cudaSuccess) e = cudaMemsetAsync(d->gdone, 0, sizeof(unsigned) * kGdoneRep * kLine, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(d->cmax, 0, sizeof(unsigned long long) * std::max<i64>(d->n, 1), s);
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
        P.pairs = d->pairs;
        P.tasks = d->tasks;
        P.gdone = d->gdone;
        P.relmap = d->relmap;
        P.phase_ptr = d->phase_ptr;
        P.n_tasks = (i32)d->n_tasks;
        P.done = d->done;
        P.cmax = d->cmax;
        P.err = err;
        P.stamps = d->stamps;
        P.trace = d->trace;
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
