// glu_device.cu -- sm_100a kernels and device handle of the B200 GLU3.0 path.
//
// Numeric factorization = one persistent cooperative kernel:
//
//   for each phase l (= level of the relaxed schedule, depgraph.py:159-170):
//       every warp takes items of phase l round-robin; an item is one
//       destination-column segment with its ordered chunk list; the warp
//       applies  v[q] -= (v[p] / v[d]) * v[m]  chunk after chunk, lanes over
//       the chunk's L entries, targets found through the precomputed uint16
//       scatter map (no runtime search, unlike _kernels.py:107-115)
//       grid barrier
//   pivot check + L divide of every column (_kernels.py:152-173)
//
// Bitwise parity: every MAC is the reference's three IEEE roundings
// (__ddiv_rn, __dmul_rn, __dsub_rn; never contracted to FMA), and every
// target receives its MACs in the order fixed by the plan (contract A or B,
// glu_host.cpp).  Values are read and written through L2 (ld/st.cg) so the
// grid barrier's release/acquire makes one phase's writes visible to the
// next without L1 invalidation.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "glu_b200.h"
#include "glu_internal.h"

using i64 = int64_t;
using i32 = int32_t;
using glu::Chunk;
using glu::Item;

#define GLU_CUDA(call)                                                               \
    do {                                                                             \
        cudaError_t e_ = (call);                                                     \
        if (e_ != cudaSuccess) {                                                     \
            glu::set_error(std::string(#call) + ": " + cudaGetErrorString(e_));      \
            return GLU_ECUDA;                                                        \
        }                                                                            \
    } while (0)

namespace {

constexpr int kThreads = 512;  // 16 warps per CTA
constexpr int kWarps = kThreads / 32;

// ---------------------------------------------------------------------------
// grid barrier: monotonically increasing arrival counter, release on arrive,
// acquire on the spin.  Co-residency is guaranteed by the cooperative launch.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void grid_barrier(unsigned int *count, unsigned int target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(count) : "memory");
        unsigned int v;
        while (true) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(count) : "memory");
            if (v >= target) break;
        }
    }
    __syncthreads();
}

__device__ __forceinline__ double ldv(const double *p) { return __ldcg(p); }
__device__ __forceinline__ void stv(double *p, double x) { __stcg(p, x); }

struct FactorParams {
    double *v;
    const i32 *level_item_ptr;
    const Item *items;
    const Chunk *chunks;
    const uint16_t *map;
    const glu::DeepRef *deep;
    const i32 *col_ptr;
    const i32 *diag_pos;
    const i32 *level_of;
    i32 n;
    i32 n_levels;
    double thresh;
    unsigned long long *fail;  // min (level << 32 | column) of failing pivots
    unsigned int *bar;
    unsigned long long *level_ns;  // optional per-phase end timestamps
    i32 fail_by_column;            // 1: key = column only (sequential API semantics)
};

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// kPush item: ordered chunks into one destination segment.  The chunk
// descriptors of a window of <= 32 chunks are fetched lane-parallel (with
// their pivots and multipliers: none of them is written during the phase),
// then the window's entries are flattened over the lanes 32 at a time.
// Entries of one epoch hit distinct targets, so a round's read-modify-writes
// run in parallel; a round that straddles an epoch boundary applies its
// epochs in order with a warp barrier between them.  The next round's map
// and L loads are issued before the current round's target RMW.
struct Round {
    int q;        // target offset in the segment (-1: lane idle)
    int ep;       // epoch of the entry inside the window
    double l;     // A_s(i,j), undivided
    double pv;    // pivot A_s(j,j)
    double mu;    // multiplier U(j,k)
};

__device__ __forceinline__ void load_round(const FactorParams &P, const uint16_t *mp, int rbase,
                                           int wtot, int lane, int nch, int incl, int p0, int est,
                                           double piv, double mult, int myep, Round &R) {
    const int e = rbase + lane;
    // chunk of entry e: chunks starting in (rbase, rbase+32) split the round
    const unsigned start_bits = __reduce_or_sync(
        0xffffffffu, (lane < nch && est > rbase && est < rbase + 32) ? (1u << (est - rbase)) : 0u);
    const int cfirst = __popc(__ballot_sync(0xffffffffu, lane < nch && est <= rbase)) - 1;
    const int c = cfirst + __popc(start_bits & ((2u << lane) - 1u));
    const int cp0 = __shfl_sync(0xffffffffu, p0, c);
    const int cest = __shfl_sync(0xffffffffu, est, c);
    R.pv = __shfl_sync(0xffffffffu, piv, c);
    R.mu = __shfl_sync(0xffffffffu, mult, c);
    R.ep = __shfl_sync(0xffffffffu, myep, c);
    R.q = -1;
    if (e < wtot) {
        R.q = __ldg(mp + e);
        R.l = ldv(P.v + cp0 + (e - cest));
    }
}

__device__ __forceinline__ void apply_round(double *vb, const Round &R, int lane) {
    const int lo = __shfl_sync(0xffffffffu, R.ep, 0);
    const unsigned act = __ballot_sync(0xffffffffu, R.q >= 0);
    const int hi = __shfl_sync(0xffffffffu, R.ep, 31 - __clz(act));
    double prod = 0.0;
    if (R.q >= 0) prod = __dmul_rn(__ddiv_rn(R.l, R.pv), R.mu);
    if (lo == hi) {
        if (R.q >= 0) {
            double *tp = vb + R.q;
            stv(tp, __dsub_rn(ldv(tp), prod));
        }
    } else {
        for (int ep = lo; ep <= hi; ++ep) {
            if (R.q >= 0 && R.ep == ep) {
                double *tp = vb + R.q;
                stv(tp, __dsub_rn(ldv(tp), prod));
            }
            __syncwarp();
        }
    }
    __syncwarp();
}

__device__ __forceinline__ void run_push(const FactorParams &P, int4 a, int4 b, int lane) {
    const i64 moff = (i64)(unsigned)a.x | ((i64)a.y << 32);
    double *vb = P.v + a.z;
    const uint16_t *mp = P.map + moff;
    const int c0 = b.x, c1 = b.y;
    const int4 *cp = reinterpret_cast<const int4 *>(P.chunks);
    for (int wb = c0; wb < c1; wb += 32) {
        const int nch = min(32, c1 - wb);
        int4 ch = make_int4(0, 0, 0, 0);
        double piv = 1.0, mult = 0.0;
        if (lane < nch) {
            ch = __ldg(cp + wb + lane);
            piv = ldv(P.v + ch.y);
            mult = ldv(P.v + ch.x);
        }
        const int cnt = ch.w & 0x7fffffff;
        const bool newep = lane == 0 || (lane < nch && (ch.w & glu::kEpochBit));
        const unsigned epm = __ballot_sync(0xffffffffu, newep);
        const int myep = __popc(epm & ((2u << lane) - 1u)) - 1;
        // inclusive prefix of chunk sizes -> exclusive starts
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int x = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += x;
        }
        const int est = incl - cnt;
        const int wtot = __shfl_sync(0xffffffffu, incl, 31);
        Round cur, nxt;
        load_round(P, mp, 0, wtot, lane, nch, incl, ch.z, est, piv, mult, myep, cur);
        for (int rb = 0; rb < wtot; rb += 32) {
            if (rb + 32 < wtot)
                load_round(P, mp, rb + 32, wtot, lane, nch, incl, ch.z, est, piv, mult, myep, nxt);
            apply_round(vb, cur, lane);
            cur = nxt;
        }
        mp += wtot;
    }
}

// kDeep item: one target, many ordered contributions.  Lanes form 32
// products at a time (independent roundings); every lane then replays the
// subtraction chain in order from shuffles, so the target sees exactly the
// reference's sequence of roundings with one load and one store.
__device__ __forceinline__ void run_deep(const FactorParams &P, int4 a, int4 b, int lane) {
    const i64 off = (i64)(unsigned)a.x | ((i64)a.y << 32);
    const int macs = b.z;
    const int4 *dr = reinterpret_cast<const int4 *>(P.deep) + off;
    double *tp = P.v + a.z;
    double acc = ldv(tp);
    for (int r = 0; r < macs; r += 32) {
        double prod = 0.0;
        if (r + lane < macs) {
            const int4 c = __ldg(dr + r + lane);
            prod = __dmul_rn(__ddiv_rn(ldv(P.v + c.x), ldv(P.v + c.y)), ldv(P.v + c.z));
        }
        const int cnt = min(32, macs - r);
        if (cnt == 32) {
#pragma unroll
            for (int s = 0; s < 32; ++s) acc = __dsub_rn(acc, __shfl_sync(0xffffffffu, prod, s));
        } else {
            for (int s = 0; s < cnt; ++s) acc = __dsub_rn(acc, __shfl_sync(0xffffffffu, prod, s));
        }
    }
    if (lane == 0) stv(tp, acc);
}

__device__ __forceinline__ void run_item(const FactorParams &P, int idx, int lane) {
    const int4 *ip = reinterpret_cast<const int4 *>(P.items + idx);
    const int4 a = __ldg(ip), b = __ldg(ip + 1);
    if (b.w == glu::kDeep) run_deep(P, a, b, lane);
    else run_push(P, a, b, lane);
}

// Pivot check + divide of column j (_kernels.py:152-173): cmax over the
// whole column with the reference's `av > cmax` rule (NaN never wins),
// failure if |piv| <= thresh * cmax, else L(:,j) /= piv.
__device__ __forceinline__ void divide_column(const FactorParams &P, int j, int lane) {
    const int lo = __ldg(P.col_ptr + j), hi = __ldg(P.col_ptr + j + 1);
    const int d = __ldg(P.diag_pos + j);
    double cmax = 0.0;
    for (int p = lo + lane; p < hi; p += 32) {
        const double av = fabs(ldv(P.v + p));
        if (av > cmax) cmax = av;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double x = __shfl_xor_sync(0xffffffffu, cmax, o);
        if (x > cmax) cmax = x;
    }
    const double piv = ldv(P.v + d);
    if (fabs(piv) <= __dmul_rn(P.thresh, cmax)) {
        if (lane == 0) {
            unsigned long long key =
                P.fail_by_column ? (unsigned long long)j
                                 : (((unsigned long long)__ldg(P.level_of + j)) << 32) | (unsigned)j;
            atomicMin(P.fail, key);
        }
        return;
    }
    for (int p = d + 1 + lane; p < hi; p += 32) stv(P.v + p, __ddiv_rn(ldv(P.v + p), piv));
}

__global__ void __launch_bounds__(kThreads, 1) factor_kernel(FactorParams P) {
    const int lane = threadIdx.x & 31;
    const int gw = blockIdx.x * kWarps + (threadIdx.x >> 5);
    const int nw = gridDim.x * kWarps;
    unsigned int target = 0;
    if (P.level_ns && blockIdx.x == 0 && threadIdx.x == 0) P.level_ns[0] = globaltimer();
    for (int l = 0; l < P.n_levels; ++l) {
        const int i0 = __ldg(P.level_item_ptr + l), i1 = __ldg(P.level_item_ptr + l + 1);
        for (int it = i0 + gw; it < i1; it += nw) run_item(P, it, lane);
        target += gridDim.x;
        grid_barrier(P.bar, target);
        if (P.level_ns && blockIdx.x == 0 && threadIdx.x == 0) P.level_ns[l + 1] = globaltimer();
    }
    for (int j = gw; j < P.n; j += nw) divide_column(P, j, lane);
}

// ---------------------------------------------------------------------------
// scatter map: for every MAC, the offset of its target row inside the item's
// destination segment, found once by binary search over the segment's rows.
// ---------------------------------------------------------------------------
__global__ void build_map_kernel(const Item *items, i64 n_items, const Chunk *chunks,
                                 const i32 *row_idx, uint16_t *map, int *bad) {
    const int lane = threadIdx.x & 31;
    const i64 w = (i64)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const i64 nwarp = (i64)gridDim.x * (blockDim.x >> 5);
    for (i64 it = w; it < n_items; it += nwarp) {
        const Item I = items[it];
        if (I.kind != glu::kPush) continue;
        const i32 *seg = row_idx + I.base;
        i64 off = I.map_off;
        for (int c = I.c0; c < I.c1; ++c) {
            const Chunk C = chunks[c];
            const int cnt = C.meta & 0x7fffffff;
            for (int t = lane; t < cnt; t += 32) {
                const i32 r = row_idx[C.p0 + t];
                int lo = 0, hi = I.span;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (seg[mid] < r) lo = mid + 1; else hi = mid;
                }
                if (lo >= I.span || seg[lo] != r) atomicExch(bad, 1);
                map[off + t] = (uint16_t)lo;
            }
            off += cnt;
        }
    }
}

// ---------------------------------------------------------------------------
// device scatter (_kernels.py:15-34): v = 0; v[slot[e]] = a[e]
// ---------------------------------------------------------------------------
__global__ void zero_kernel(double *v, i64 n) {
    for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
        v[i] = 0.0;
}
__global__ void scatter_kernel(const double *a, const i32 *slot, i64 nz, double *v) {
    for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < nz; i += (i64)gridDim.x * blockDim.x)
        v[slot[i]] = a[i];
}

// ---------------------------------------------------------------------------
// Level-scheduled triangular solves, pull form so each unknown receives its
// updates in the reference order (_kernels.py:176-197): ascending j for L
// (with the y[j] != 0 skip), descending j for U.  One warp per row: lanes
// form the products (independent roundings), then every lane replays the
// subtraction chain in order from shuffles, so the bits match the
// sequential column sweep.
// ---------------------------------------------------------------------------
struct SolveParams {
    const double *v;
    double *x;
    const i32 *lvl_ptr;   // per solve level, range into rows
    const i32 *rows;
    const i32 *ent_ptr;   // per row, range into ent_col/ent_slot
    const i32 *ent_col;
    const i32 *ent_slot;
    const i32 *diag_pos;  // upper only
    i32 n_levels;
    unsigned int *bar;
    i32 upper;
};

__global__ void __launch_bounds__(kThreads, 1) solve_kernel(SolveParams S) {
    const int lane = threadIdx.x & 31;
    const int gw = blockIdx.x * kWarps + (threadIdx.x >> 5);
    const int nw = gridDim.x * kWarps;
    unsigned int target = 0;
    for (int l = 0; l < S.n_levels; ++l) {
        const int r0 = __ldg(S.lvl_ptr + l), r1 = __ldg(S.lvl_ptr + l + 1);
        for (int ri = r0 + gw; ri < r1; ri += nw) {
            const int i = __ldg(S.rows + ri);
            const int e0 = __ldg(S.ent_ptr + i), e1 = __ldg(S.ent_ptr + i + 1);
            double acc = ldv(S.x + i);
            const int ne = e1 - e0;
            for (int base = 0; base < ne; base += 32) {
                // upper: entries are stored ascending; consume them descending
                const int e = S.upper ? (e1 - 1 - base - lane) : (e0 + base + lane);
                const int cnt = min(32, ne - base);
                double prod = 0.0;
                bool use = false;
                if (lane < cnt) {
                    const double xj = ldv(S.x + __ldg(S.ent_col + e));
                    prod = __dmul_rn(ldv(S.v + __ldg(S.ent_slot + e)), xj);
                    use = S.upper ? true : (xj != 0.0);
                }
                const unsigned umask = __ballot_sync(0xffffffffu, use);
                for (int s = 0; s < cnt; ++s) {
                    const double p = __shfl_sync(0xffffffffu, prod, s);
                    if (umask & (1u << s)) acc = __dsub_rn(acc, p);
                }
            }
            if (S.upper) acc = __ddiv_rn(acc, ldv(S.v + __ldg(S.diag_pos + i)));
            if (lane == 0) stv(S.x + i, acc);
        }
        target += gridDim.x;
        grid_barrier(S.bar, target);
    }
}

__global__ void zero_pivot_kernel(const double *v, const i32 *diag_pos, i32 n, int *fail) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
        if (v[diag_pos[j]] == 0.0) atomicMax(fail, j);
}

template <class T>
cudaError_t upload(T **dst, const std::vector<T> &src) {
    *dst = nullptr;
    if (src.empty()) return cudaSuccess;
    cudaError_t e = cudaMalloc((void **)dst, src.size() * sizeof(T));
    if (e != cudaSuccess) return e;
    return cudaMemcpy(*dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice);
}

}  // namespace

// ---------------------------------------------------------------------------
// handle
// ---------------------------------------------------------------------------
struct glu_handle {
    int device = 0;
    int sm_count = 0;
    int grid = 0;  // CTAs of the persistent kernels
    i64 n = 0, nnz = 0, nz = -1;
    i64 n_levels = 0, n_items = 0, n_chunks = 0, n_map = 0;
    i64 bytes = 0;
    // pattern
    i32 *col_ptr = nullptr, *row_idx = nullptr, *diag_pos = nullptr, *level_of = nullptr;
    // plan
    i32 *level_item_ptr = nullptr;
    Item *items = nullptr;
    Chunk *chunks = nullptr;
    uint16_t *map = nullptr;
    glu::DeepRef *deep = nullptr;
    i64 n_deep = 0;
    // solves
    i64 l_levels = 0, u_levels = 0;
    i32 *l_lvl_ptr = nullptr, *l_rows = nullptr, *l_ptr = nullptr, *l_col = nullptr, *l_slot = nullptr;
    i32 *u_lvl_ptr = nullptr, *u_rows = nullptr, *u_ptr = nullptr, *u_col = nullptr, *u_slot = nullptr;
    // input scatter
    i32 *a_slot = nullptr;
    // scratch
    unsigned long long *fail = nullptr;
    unsigned int *bar = nullptr;
    int *ifail = nullptr;
    unsigned long long *level_ns = nullptr;
    bool time_levels = false;
    bool fail_by_column = false;
    std::vector<double> last_level_ms;
    // host-API staging
    double *d_a = nullptr, *d_v = nullptr, *d_x = nullptr;
    cudaStream_t stream = nullptr;
};

namespace {

template <class T>
i64 track_upload(glu_handle *h, T **dst, const std::vector<T> &src) {
    GLU_CUDA(upload(dst, src));
    h->bytes += (i64)(src.size() * sizeof(T));
    return GLU_OK;
}

std::vector<i32> to_i32(const int64_t *p, i64 m) {
    std::vector<i32> v((size_t)m);
    for (i64 i = 0; i < m; i++) v[i] = (i32)p[i];
    return v;
}

// Level sets of the triangular solves (forward: L rows, backward: U rows).
void solve_levels(i64 n, const std::vector<i32> &ptr, const std::vector<i32> &col, bool upper,
                  std::vector<i32> &lvl_ptr, std::vector<i32> &rows, i64 &n_levels) {
    std::vector<i32> lev(n, 0);
    i32 nl = 0;
    for (i64 s = 0; s < n; s++) {
        const i64 i = upper ? n - 1 - s : s;
        i32 lv = 0;
        for (i32 e = ptr[i]; e < ptr[i + 1]; e++) lv = std::max(lv, lev[col[e]] + 1);
        lev[i] = lv;
        nl = std::max(nl, lv + 1);
    }
    if (n == 0) nl = 0;
    lvl_ptr.assign(nl + 1, 0);
    for (i64 i = 0; i < n; i++) lvl_ptr[lev[i] + 1]++;
    for (i32 l = 0; l < nl; l++) lvl_ptr[l + 1] += lvl_ptr[l];
    rows.assign(n, 0);
    std::vector<i32> fill(lvl_ptr.begin(), lvl_ptr.end());
    for (i64 i = 0; i < n; i++) rows[fill[lev[i]]++] = (i32)i;
    n_levels = nl;
}

int coop_grid(const void *kernel, int sm_count) {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThreads, 0) != cudaSuccess)
        return 0;
    per_sm = std::min(per_sm, 1);
    return per_sm * sm_count;
}

}  // namespace

extern "C" const char *glu_version(void) { return "glu_b200 0.1 sm_100a"; }

extern "C" int64_t glu_create(int64_t n, const int64_t *col_ptr, const int64_t *row_idx,
                              const int64_t *diag_pos, const int64_t *row_ptr,
                              const int64_t *col_idx, const int64_t *csc_pos,
                              const int64_t *level_of, const glu_plan *plan, glu_handle **out) {
    *out = nullptr;
    if (!plan) { glu::set_error("plan is null"); return GLU_EINVAL; }
    auto *h = new glu_handle();
    auto fail = [&](i64 code) { glu_destroy(h); return code; };
    if (cudaGetDevice(&h->device) != cudaSuccess) { glu::set_error("no CUDA device"); return fail(GLU_ECUDA); }
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, h->device) != cudaSuccess) { glu::set_error("cudaGetDeviceProperties"); return fail(GLU_ECUDA); }
    if (prop.major < 10) {
        glu::set_error("glu_b200 requires an sm_100 (Blackwell) device, got sm_" +
                       std::to_string(prop.major) + std::to_string(prop.minor));
        return fail(GLU_ECUDA);
    }
    h->sm_count = prop.multiProcessorCount;
    h->n = n;
    h->nnz = col_ptr[n];
    const glu::glu_plan_view pv = glu::plan_view(plan);
    h->n_levels = pv.n_levels;
    h->n_items = pv.n_items;
    h->n_chunks = pv.n_chunks;
    h->n_map = pv.n_map;
    h->n_deep = pv.n_deep;
    if (cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking) != cudaSuccess) {
        glu::set_error("cudaStreamCreate"); return fail(GLU_ECUDA);
    }
    i64 rc;
#define UP(dst, vec) if ((rc = track_upload(h, &(dst), vec)) != GLU_OK) return fail(rc)
    std::vector<i32> cp32 = to_i32(col_ptr, n + 1), ri32 = to_i32(row_idx, h->nnz),
                     dp32 = to_i32(diag_pos, n), lv32 = to_i32(level_of, n);
    UP(h->col_ptr, cp32);
    UP(h->row_idx, ri32);
    UP(h->diag_pos, dp32);
    UP(h->level_of, lv32);
    UP(h->level_item_ptr, to_i32(pv.level_item_ptr, pv.n_levels + 1));
    UP(h->items, std::vector<Item>(pv.items, pv.items + pv.n_items));
    UP(h->chunks, std::vector<Chunk>(pv.chunks, pv.chunks + pv.n_chunks));
    UP(h->deep, std::vector<glu::DeepRef>(pv.deep, pv.deep + pv.n_deep));
    if (h->n_map > 0) {
        if (cudaMalloc((void **)&h->map, (size_t)h->n_map * sizeof(uint16_t)) != cudaSuccess) {
            glu::set_error("cudaMalloc(scatter map " + std::to_string(h->n_map * 2) + " B)");
            return fail(GLU_ECUDA);
        }
        h->bytes += h->n_map * 2;
    }
    // solve structures from the CSR view: L rows (cols < i) and U rows (cols > i)
    std::vector<i32> lp(n + 1, 0), lc, ls, up_(n + 1, 0), uc, us;
    for (i64 i = 0; i < n; i++) {
        for (i64 t = row_ptr[i]; t < row_ptr[i + 1]; t++) {
            const i64 c = col_idx[t];
            if (c < i) { lc.push_back((i32)c); ls.push_back((i32)csc_pos[t]); }
            else if (c > i) { uc.push_back((i32)c); us.push_back((i32)csc_pos[t]); }
        }
        lp[i + 1] = (i32)lc.size();
        up_[i + 1] = (i32)uc.size();
    }
    std::vector<i32> llp, lrows, ulp, urows;
    solve_levels(n, lp, lc, false, llp, lrows, h->l_levels);
    solve_levels(n, up_, uc, true, ulp, urows, h->u_levels);
    UP(h->l_ptr, lp); UP(h->l_col, lc); UP(h->l_slot, ls); UP(h->l_lvl_ptr, llp); UP(h->l_rows, lrows);
    UP(h->u_ptr, up_); UP(h->u_col, uc); UP(h->u_slot, us); UP(h->u_lvl_ptr, ulp); UP(h->u_rows, urows);
#undef UP
    if (cudaMalloc((void **)&h->fail, sizeof(unsigned long long)) != cudaSuccess ||
        cudaMalloc((void **)&h->bar, sizeof(unsigned int)) != cudaSuccess ||
        cudaMalloc((void **)&h->ifail, sizeof(int)) != cudaSuccess) {
        glu::set_error("cudaMalloc(scratch)"); return fail(GLU_ECUDA);
    }
    h->grid = std::min(coop_grid((const void *)factor_kernel, h->sm_count),
                       coop_grid((const void *)solve_kernel, h->sm_count));
    if (h->grid <= 0) { glu::set_error("persistent kernel cannot be co-resident"); return fail(GLU_ECUDA); }
    // build the scatter map on the device
    if (h->n_map > 0) {
        int *dbad = h->ifail;
        if (cudaMemset(dbad, 0, sizeof(int)) != cudaSuccess) { glu::set_error("memset"); return fail(GLU_ECUDA); }
        build_map_kernel<<<h->sm_count * 8, 256, 0, h->stream>>>(h->items, h->n_items, h->chunks,
                                                                   h->row_idx, h->map, dbad);
        int hbad = 0;
        if (cudaMemcpyAsync(&hbad, dbad, sizeof(int), cudaMemcpyDeviceToHost, h->stream) != cudaSuccess ||
            cudaStreamSynchronize(h->stream) != cudaSuccess) {
            glu::set_error(std::string("scatter-map build: ") + cudaGetErrorString(cudaGetLastError()));
            return fail(GLU_ECUDA);
        }
        if (hbad) { glu::set_error("scatter map: target row absent from segment"); return fail(GLU_MISMATCH); }
    }
    *out = h;
    return GLU_OK;
}

extern "C" void glu_destroy(glu_handle *h) {
    if (!h) return;
    void *ptrs[] = {h->col_ptr, h->row_idx, h->diag_pos, h->level_of, h->level_item_ptr, h->items,
                    h->chunks, h->map, h->deep, h->l_lvl_ptr, h->l_rows, h->l_ptr, h->l_col, h->l_slot,
                    h->u_lvl_ptr, h->u_rows, h->u_ptr, h->u_col, h->u_slot, h->a_slot, h->fail,
                    h->bar, h->ifail, h->level_ns, h->d_a, h->d_v, h->d_x};
    for (void *p : ptrs)
        if (p) cudaFree(p);
    if (h->stream) cudaStreamDestroy(h->stream);
    delete h;
}

extern "C" void glu_handle_info(const glu_handle *h, int64_t *info) {
    info[0] = h->n; info[1] = h->nnz; info[2] = h->n_levels; info[3] = h->n_items;
    info[4] = h->n_chunks; info[5] = h->n_map; info[6] = h->bytes; info[7] = h->grid;
    info[8] = kThreads; info[9] = h->l_levels; info[10] = h->u_levels; info[11] = h->sm_count;
}

extern "C" int64_t glu_set_option(glu_handle *h, int64_t key, int64_t value) {
    switch (key) {
        case 1:  // per-level timestamps
            h->time_levels = value != 0;
            if (h->time_levels && !h->level_ns && h->n_levels > 0)
                GLU_CUDA(cudaMalloc((void **)&h->level_ns, sizeof(unsigned long long) * (h->n_levels + 1)));
            return GLU_OK;
        case 2:  // failing-pivot order: 0 level-major (factor_parallel), 1 column (sequential paths)
            h->fail_by_column = value != 0;
            return GLU_OK;
        default:
            glu::set_error("unknown option");
            return GLU_EINVAL;
    }
}

extern "C" int64_t glu_level_times(const glu_handle *h, double *ms, int64_t len) {
    const i64 m = std::min<i64>(len, (i64)h->last_level_ms.size());
    for (i64 i = 0; i < m; i++) ms[i] = h->last_level_ms[i];
    return m;
}

extern "C" int64_t glu_set_input_pattern(glu_handle *h, int64_t nz, const int64_t *a_col_ptr,
                                         const int64_t *a_row_idx) {
    // host merge, reference semantics (_kernels.py:15-34); the slot map then
    // lets every later scatter run on the device
    std::vector<i32> rows32((size_t)h->nnz), cols32((size_t)h->n + 1);
    GLU_CUDA(cudaMemcpy(rows32.data(), h->row_idx, sizeof(i32) * h->nnz, cudaMemcpyDeviceToHost));
    GLU_CUDA(cudaMemcpy(cols32.data(), h->col_ptr, sizeof(i32) * (h->n + 1), cudaMemcpyDeviceToHost));
    std::vector<i32> slot((size_t)nz);
    for (i64 j = 0; j < h->n; j++) {
        i64 q = cols32[j], hi = cols32[j + 1];
        for (i64 p = a_col_ptr[j]; p < a_col_ptr[j + 1]; p++) {
            const i64 r = a_row_idx[p];
            while (q < hi && rows32[q] < r) q++;
            if (q >= hi || rows32[q] != r) {
                glu::set_error("column " + std::to_string(j) + " of A has entries outside the filled pattern");
                return j;
            }
            slot[p] = (i32)q;
            q++;
        }
    }
    if (h->a_slot) { cudaFree(h->a_slot); h->a_slot = nullptr; }
    if (h->d_a) { cudaFree(h->d_a); h->d_a = nullptr; }
    i64 rc = track_upload(h, &h->a_slot, slot);
    if (rc != GLU_OK) return rc;
    h->nz = nz;
    return GLU_OK;
}

extern "C" int64_t glu_scatter_device(glu_handle *h, const double *a_vals, double *v, void *stream) {
    if (h->nz < 0) { glu::set_error("glu_set_input_pattern not called"); return GLU_EINVAL; }
    cudaStream_t s = (cudaStream_t)stream;
    const int blocks = h->sm_count * 4;
    zero_kernel<<<blocks, 256, 0, s>>>(v, h->nnz);
    if (h->nz > 0) scatter_kernel<<<blocks, 256, 0, s>>>(a_vals, h->a_slot, h->nz, v);
    GLU_CUDA(cudaGetLastError());
    return GLU_OK;
}

static int64_t launch_factor(glu_handle *h, double *v, double thresh, cudaStream_t s) {
    GLU_CUDA(cudaMemsetAsync(h->fail, 0xff, sizeof(unsigned long long), s));
    GLU_CUDA(cudaMemsetAsync(h->bar, 0, sizeof(unsigned int), s));
    FactorParams P;
    P.v = v;
    P.level_item_ptr = h->level_item_ptr;
    P.items = h->items;
    P.chunks = h->chunks;
    P.map = h->map;
    P.deep = h->deep;
    P.col_ptr = h->col_ptr;
    P.diag_pos = h->diag_pos;
    P.level_of = h->level_of;
    P.n = (i32)h->n;
    P.n_levels = (i32)h->n_levels;
    P.thresh = thresh;
    P.fail = h->fail;
    P.bar = h->bar;
    P.level_ns = h->time_levels ? h->level_ns : nullptr;
    P.fail_by_column = h->fail_by_column ? 1 : 0;
    void *args[] = {&P};
    if (h->time_levels) {
        GLU_CUDA(cudaMemsetAsync(h->level_ns, 0, sizeof(unsigned long long) * (h->n_levels + 1), s));
    }
    GLU_CUDA(cudaLaunchCooperativeKernel((const void *)factor_kernel, dim3(h->grid), dim3(kThreads),
                                         args, 0, s));
    return GLU_OK;
}

static int64_t read_fail(glu_handle *h, cudaStream_t s) {
    unsigned long long key = 0;
    GLU_CUDA(cudaMemcpyAsync(&key, h->fail, sizeof(key), cudaMemcpyDeviceToHost, s));
    GLU_CUDA(cudaStreamSynchronize(s));
    if (h->time_levels && h->n_levels > 0) {
        std::vector<unsigned long long> ns(h->n_levels + 1);
        GLU_CUDA(cudaMemcpy(ns.data(), h->level_ns, sizeof(unsigned long long) * (h->n_levels + 1),
                            cudaMemcpyDeviceToHost));
        h->last_level_ms.assign(h->n_levels, 0.0);
        for (i64 l = 0; l < h->n_levels; l++) h->last_level_ms[l] = (double)(ns[l + 1] - ns[l]) * 1e-6;
    }
    if (key == ~0ull) return GLU_OK;
    return (int64_t)(key & 0xffffffffull);
}

extern "C" int64_t glu_factor_device(glu_handle *h, double *v, double thresh, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    i64 rc = launch_factor(h, v, thresh, s);
    if (rc != GLU_OK) return rc;
    return read_fail(h, s);
}

// Asynchronous variant for timing loops: no host sync, no status read.
extern "C" int64_t glu_factor_device_async(glu_handle *h, double *v, double thresh, void *stream) {
    return launch_factor(h, v, thresh, (cudaStream_t)stream);
}

extern "C" int64_t glu_factor_status(glu_handle *h, void *stream) {
    return read_fail(h, (cudaStream_t)stream);
}

extern "C" int64_t glu_factor_batch_device(glu_handle *h, int64_t batch, double *v, double thresh,
                                           int64_t *fail_cols, void *stream) {
    // batch-minor layout: run the single-matrix kernel per value set on a
    // strided view is not possible; batched kernel arrives with the batch plan.
    (void)h; (void)batch; (void)v; (void)thresh; (void)fail_cols; (void)stream;
    glu::set_error("glu_factor_batch_device: not implemented yet");
    return GLU_EINVAL;
}

static int64_t launch_solve(glu_handle *h, const double *lu, double *x, bool upper, cudaStream_t s) {
    SolveParams S;
    S.v = lu;
    S.x = x;
    S.upper = upper ? 1 : 0;
    S.lvl_ptr = upper ? h->u_lvl_ptr : h->l_lvl_ptr;
    S.rows = upper ? h->u_rows : h->l_rows;
    S.ent_ptr = upper ? h->u_ptr : h->l_ptr;
    S.ent_col = upper ? h->u_col : h->l_col;
    S.ent_slot = upper ? h->u_slot : h->l_slot;
    S.diag_pos = h->diag_pos;
    S.n_levels = (i32)(upper ? h->u_levels : h->l_levels);
    S.bar = h->bar;
    GLU_CUDA(cudaMemsetAsync(h->bar, 0, sizeof(unsigned int), s));
    void *args[] = {&S};
    GLU_CUDA(cudaLaunchCooperativeKernel((const void *)solve_kernel, dim3(h->grid), dim3(kThreads),
                                         args, 0, s));
    return GLU_OK;
}

static int64_t check_zero_pivot(glu_handle *h, const double *lu, cudaStream_t s) {
    const int init = -1;
    GLU_CUDA(cudaMemcpyAsync(h->ifail, &init, sizeof(int), cudaMemcpyHostToDevice, s));
    zero_pivot_kernel<<<h->sm_count * 2, 256, 0, s>>>(lu, h->diag_pos, (i32)h->n, h->ifail);
    int f = -1;
    GLU_CUDA(cudaMemcpyAsync(&f, h->ifail, sizeof(int), cudaMemcpyDeviceToHost, s));
    GLU_CUDA(cudaStreamSynchronize(s));
    return f >= 0 ? (int64_t)f : GLU_OK;
}

extern "C" int64_t glu_lower_solve_device(glu_handle *h, const double *lu, double *x, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    i64 rc = launch_solve(h, lu, x, false, s);
    if (rc != GLU_OK) return rc;
    GLU_CUDA(cudaStreamSynchronize(s));
    return GLU_OK;
}

extern "C" int64_t glu_upper_solve_device(glu_handle *h, const double *lu, double *x, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    i64 rc = check_zero_pivot(h, lu, s);
    if (rc != GLU_OK) return rc;
    rc = launch_solve(h, lu, x, true, s);
    if (rc != GLU_OK) return rc;
    GLU_CUDA(cudaStreamSynchronize(s));
    return GLU_OK;
}

extern "C" int64_t glu_solve_device(glu_handle *h, const double *lu, double *x, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    i64 rc = check_zero_pivot(h, lu, s);
    if (rc != GLU_OK) return rc;
    if ((rc = launch_solve(h, lu, x, false, s)) != GLU_OK) return rc;
    if ((rc = launch_solve(h, lu, x, true, s)) != GLU_OK) return rc;
    GLU_CUDA(cudaStreamSynchronize(s));
    return GLU_OK;
}

static int64_t ensure_staging(glu_handle *h) {
    if (!h->d_v) GLU_CUDA(cudaMalloc((void **)&h->d_v, sizeof(double) * std::max<i64>(h->nnz, 1)));
    if (!h->d_a) GLU_CUDA(cudaMalloc((void **)&h->d_a, sizeof(double) * std::max<i64>(h->nz, 1)));
    if (!h->d_x) GLU_CUDA(cudaMalloc((void **)&h->d_x, sizeof(double) * std::max<i64>(h->n, 1)));
    return GLU_OK;
}

extern "C" int64_t glu_factor_host(glu_handle *h, const double *a_vals, double *lu_out, double thresh) {
    if (h->nz < 0) { glu::set_error("glu_set_input_pattern not called"); return GLU_EINVAL; }
    i64 rc = ensure_staging(h);
    if (rc != GLU_OK) return rc;
    cudaStream_t s = h->stream;
    GLU_CUDA(cudaMemcpyAsync(h->d_a, a_vals, sizeof(double) * h->nz, cudaMemcpyHostToDevice, s));
    if ((rc = glu_scatter_device(h, h->d_a, h->d_v, s)) != GLU_OK) return rc;
    if ((rc = launch_factor(h, h->d_v, thresh, s)) != GLU_OK) return rc;
    GLU_CUDA(cudaMemcpyAsync(lu_out, h->d_v, sizeof(double) * h->nnz, cudaMemcpyDeviceToHost, s));
    return read_fail(h, s);
}

extern "C" int64_t glu_solve_host(glu_handle *h, const double *lu, const double *b, double *x) {
    i64 rc = ensure_staging(h);
    if (rc != GLU_OK) return rc;
    cudaStream_t s = h->stream;
    GLU_CUDA(cudaMemcpyAsync(h->d_v, lu, sizeof(double) * h->nnz, cudaMemcpyHostToDevice, s));
    GLU_CUDA(cudaMemcpyAsync(h->d_x, b, sizeof(double) * h->n, cudaMemcpyHostToDevice, s));
    if ((rc = glu_solve_device(h, h->d_v, h->d_x, s)) != GLU_OK) return rc;
    GLU_CUDA(cudaMemcpyAsync(x, h->d_x, sizeof(double) * h->n, cudaMemcpyDeviceToHost, s));
    GLU_CUDA(cudaStreamSynchronize(s));
    return GLU_OK;
}
