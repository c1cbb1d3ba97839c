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
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
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
constexpr int kLineWords = 32;   // u32 stride between hot words (one 128 B line each)
constexpr int kColRep = 4;       // replicas of each column's completion counter (spread the pollers)
constexpr unsigned long long kWatchdogNs = 4000000000ull;  // 4 s: a dependency wait this long is a bug

// L2 residency: the plan streams (items, chunks, maps, deep refs: ~1 GB for
// cfg2, read once per factorization) are loaded with an evict_first policy so
// they do not push the 34 MB value array out of the 126 MB L2; the values
// themselves use plain .cg accesses (L2, the coherence point for the
// dataflow sync).  An evict_last policy on the values measured slightly
// slower (cfg2: 6.57 vs 6.51 ms): they stay resident either way.
__device__ __forceinline__ uint64_t pol_first() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ double ldv(const double *p) { return __ldcg(p); }
__device__ __forceinline__ void stv(double *p, double x) { __stcg(p, x); }
// read-only plan streams
__device__ __forceinline__ int4 ldp(const int4 *p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p), "l"(pol_first()));
    return r;
}
__device__ __forceinline__ int ldp8(const uint8_t *p) {
    unsigned short r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u8 %0, [%1], %2;"
                 : "=h"(r) : "l"(p), "l"(pol_first()));
    return (int)r;
}
__device__ __forceinline__ int ldp16(const uint16_t *p) {
    unsigned short r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u16 %0, [%1], %2;"
                 : "=h"(r) : "l"(p), "l"(pol_first()));
    return (int)r;
}

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
struct FactorParams {
    double *v;
    const Item *items;
    const Chunk *chunks;
    const uint8_t *map8;
    const uint16_t *tgt16;
    const glu::DeepRef *deep;
    const i32 *col_ptr;
    const i32 *diag_pos;
    const i32 *level_of;
    const i32 *level_need;  // items per phase
    i32 n;
    i32 n_items;
    i32 n_levels;
    i32 n_div;              // columns the final pass divides (the dense tail divides its own)
    i32 nb;                 // value sets factored by this launch (batch-major, set_stride apart)
    long long set_stride;
    double thresh;
    unsigned long long *fail;  // per value set: min (level << 32 | column) of failing pivots
    unsigned *done;            // per phase: completed items (stride 8 words)
    unsigned *col_done;        // per column: completed items into it
    const i32 *col_total;      // per column: items into it
    const glu::ColDep *cdeps;  // per item: destination columns + earlier-phase counts
    int *err;                  // watchdog flag
    unsigned long long *level_ns;  // optional per-phase completion timestamps
    unsigned long long *trace;     // optional per-item timestamps (diagnostics)
    i32 trace_i0, trace_i1;        // traced item range
    i32 poll_ns;                   // sleep between dependency polls
    i32 fail_by_column;            // 1: key = column only (sequential API semantics)
};

// ---------------------------------------------------------------------------
// Dataflow synchronisation (replaces a grid barrier per level).
//
// Items are ordered by phase and dealt round-robin to the warps; a warp runs
// its items in order and, on entering phase l, waits until every phase < l
// is complete -- a point-to-point wait instead of a grid-wide barrier, so a
// warp with nothing to do in phase l runs ahead to its next item and loads
// its static plan data early.
//   producer  when a warp leaves phase l it adds the number of items it ran
//             there to done[l]: fence.acq_rel + fire-and-forget red.add.
//   consumer  each CTA keeps `known` in shared memory = the number of
//             leading phases known complete.  At most one warp per CTA polls
//             at a time: lanes read done[known .. known+31] (relaxed) in one
//             round trip, compare with the static item counts and advance
//             `known` over the complete prefix (phases without items are
//             complete by definition), then fence.acq_rel.  The other warps
//             of the CTA spin on shared memory.
// No deadlock: the smallest unfinished item's warp has finished all its
// earlier items and every item it waits on has a smaller index.  A
// watchdog turns an endless wait (a bug) into an error instead of a hang.
// ---------------------------------------------------------------------------
constexpr int kReq = 4;  // dependency requests per waiting warp (distinct columns)
struct CtaSync {
    unsigned known;   // phases [0, known) complete
    int polling;      // a warp of this CTA has a poll in flight
    // per-CTA wait service (see wait_cols)
    int req_col[kWarps * kReq];
    unsigned req_need[kWarps * kReq];
    int pending[kWarps];  // 1: the warp's requests await checking
    int ready[kWarps];    // 1: all of the warp's requests satisfied
    int wpoll;            // a warp is running the service round
};

__device__ __forceinline__ unsigned ld_relaxed(const unsigned *p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void red_add_relaxed(unsigned *p, unsigned x) {
    asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(x) : "memory");
}

// wait until phases [0, w] are complete
__device__ __noinline__ bool wait_phase_impl(const unsigned *done, const i32 *level_need, int n_levels,
                                             int *err, int w, int lane, CtaSync *cs) {
    const unsigned target = (unsigned)w + 1;
    unsigned long long t0 = 0;
    volatile unsigned *vk = &cs->known;
    for (int spin = 0;; ++spin) {
        if (*vk >= target) break;
        int got = 0;
        if (lane == 0) got = atomicCAS(&cs->polling, 0, 1) == 0;
        got = __shfl_sync(0xffffffffu, got, 0);
        if (got) {
            const unsigned k0 = *vk;
            const unsigned k = k0 + lane;
            bool ok = true;
            if (k < (unsigned)n_levels) ok = ld_relaxed(done + (size_t)k * 8) >= (unsigned)__ldg(level_need + k);
            const unsigned bad = __ballot_sync(0xffffffffu, !ok);
            const unsigned adv = bad ? __ffs(bad) - 1 : 32;
            if (lane == 0) {
                fence_acq_rel_gpu();
                if (adv) atomicMax(&cs->known, k0 + adv);
                atomicExch(&cs->polling, 0);
            }
            __syncwarp();
            if (k0 + adv >= target) break;
        } else {
            __nanosleep(32);
        }
        if ((spin & 255) == 255) {
            int bad = 0;
            if (lane == 0) {
                const unsigned long long t = globaltimer();
                if (t0 == 0) t0 = t;
                bad = (t - t0 > kWatchdogNs) || *(volatile int *)err;
                if (bad) atomicExch(err, 1);
            }
            if (__shfl_sync(0xffffffffu, bad, 0)) return false;
        }
    }
    if (lane == 0) asm volatile("fence.acq_rel.cta;" ::: "memory");
    __syncwarp();
    return true;
}

__device__ __forceinline__ bool wait_phase(const FactorParams &P, int w, int lane, CtaSync *cs) {
    return wait_phase_impl(P.done, P.level_need, P.n_levels, P.err, w, lane, cs);
}

// Item completion.  A consumer of column k waits until every item into k
// is counted in col_done[k]; a counted item's stores must be visible first
// (fence.acq_rel.gpu, then the count).  Fences are expensive (~300 ns), so a
// warp batches: the item into a column that the NEXT phase reads as a source
// ("critical", the chain of the deep tail) is released at once; the others
// queue in shared memory and are released together when the warp leaves the
// phase (or the queue is full) -- never later than the phase counter, so the
// dependency order and the deadlock-freedom argument are unchanged.
constexpr int kMaxCols = 4;  // destination columns per item (glu_host.cpp kMaxItemCols)
struct WarpQ {
    int col[32];
};

__device__ __forceinline__ void flush_items(const FactorParams &P, WarpQ *q, int &nq, int lvl,
                                            unsigned ran, bool phase_end, int lane) {
    __syncwarp();
    fence_acq_rel_gpu();
    for (int x = lane; x < nq * kColRep; x += 32)
        red_add_relaxed(P.col_done + (size_t)q->col[x / kColRep] * kColRep + (x % kColRep), 1);
    if (phase_end && lane == 0) {
        unsigned *ctr = P.done + (size_t)lvl * 8;
        if (P.level_ns) {
            const unsigned old = atomicAdd(ctr, ran);
            if (old + ran == (unsigned)__ldg(P.level_need + lvl)) P.level_ns[lvl + 1] = globaltimer();
        } else {
            red_add_relaxed(ctr, ran);
        }
    }
    nq = 0;
    __syncwarp();
}

__device__ __forceinline__ void finish_item(const FactorParams &P, WarpQ *q, int &nq, int mycol,
                                            int ncol, bool crit, int lvl, unsigned ran,
                                            bool phase_end, int lane) {
    // lanes < ncol hold the item's destination columns in mycol
    if (crit) {
        const int cc = __shfl_sync(0xffffffffu, mycol, (lane / kColRep) & 31);
        __syncwarp();
        fence_acq_rel_gpu();
        if (lane < ncol * kColRep) red_add_relaxed(P.col_done + (size_t)cc * kColRep + (lane % kColRep), 1);
    } else {
        if (lane < ncol) q->col[nq + lane] = mycol;
        nq += ncol;
    }
    if (phase_end || nq + kMaxCols > 32) flush_items(P, q, nq, lvl, ran, phase_end, lane);
}

// Fine-grained wait of a push item in phase lvl: its source columns complete
// (every item into them counted) and every earlier-phase item into its own
// column counted.  Skipped when the CTA already knows phases < lvl complete.
//
// A per-CTA wait service keeps the polling off the critical path: a release
// fence (MEMBAR.GPU) waits behind every memory request the SM has in flight
// (measured: ~265 cycles on a quiet SM, ~1,500-1,900 with neighbour warps
// polling), so instead of each waiting warp polling global counters, a
// warp posts its <= kReq (column, count) requests in shared memory and ONE
// warp of the CTA at a time checks every posted request in a single round
// of relaxed loads, flagging the satisfied warps.  Relaxed polling is
// enough: the values are read .cg from L2 after the wait, and the producer
// fenced its stores before counting.
__device__ __forceinline__ bool wait_cols(const FactorParams &P, int lane, bool has_src, int j,
                                          unsigned jneed, bool has_own, int k, unsigned kneed,
                                          int lvl, CtaSync *cs, int rep) {
    const int w = threadIdx.x >> 5;
    volatile int *vready = cs->ready;
    volatile unsigned *vk = &cs->known;
    // distinct requests: the own columns (lanes < ncol, distinct by
    // construction) and every distinct source column
    const unsigned same = __match_any_sync(0xffffffffu, has_src ? j : -1 - lane);
    const bool src_lead = has_src && (__ffs(same) - 1) == lane;
    const unsigned om = __ballot_sync(0xffffffffu, has_own);
    const unsigned pm = __ballot_sync(0xffffffffu, src_lead);
    const int nown = __popc(om), nsrc = __popc(pm);
    unsigned long long t0 = 0;
    if (nown + nsrc <= kReq) {
        if (has_own) {
            const int slot = __popc(om & ((1u << lane) - 1u));
            cs->req_col[w * kReq + slot] = k;
            cs->req_need[w * kReq + slot] = kneed;
        }
        if (src_lead) {
            const int slot = nown + __popc(pm & ((1u << lane) - 1u));
            cs->req_col[w * kReq + slot] = j;
            cs->req_need[w * kReq + slot] = jneed;
        }
        if (lane == 0)
            for (int x = nown + nsrc; x < kReq; ++x) cs->req_col[w * kReq + x] = -1;
        __syncwarp();
        if (lane == 0) { cs->ready[w] = 0; __threadfence_block(); cs->pending[w] = 1; }
        __syncwarp();
        // only the service round clears a posted request (no other exit), so a
        // round never sees a half-rewritten request
        for (int spin = 0;; ++spin) {
            if (vready[w]) break;
            int got = 0;
            if (lane == 0) got = atomicCAS(&cs->wpoll, 0, 1) == 0;
            got = __shfl_sync(0xffffffffu, got, 0);
            if (got) {
                // one service round: lanes over (warp, slot) entries, two per
                // lane; the group leader's single read of pending[] decides for
                // all four lanes of a warp's entries (a request posted during
                // the round is left for the next one)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int e = lane + 32 * h, ww = e / kReq;
                    int pend = 0;
                    if ((lane % kReq) == 0) pend = ((volatile int *)cs->pending)[ww];
                    pend = __shfl_sync(0xffffffffu, pend, lane & ~(kReq - 1));
                    bool ok = true;
                    if (pend) {
                        const int cc = ((volatile int *)cs->req_col)[e];
                        if (cc >= 0)
                            ok = ld_relaxed(P.col_done + (size_t)cc * kColRep + rep) >=
                                 ((volatile unsigned *)cs->req_need)[e];
                    }
                    const unsigned bad = __ballot_sync(0xffffffffu, !ok);
                    if ((lane % kReq) == 0 && pend && ((bad >> lane) & ((1u << kReq) - 1u)) == 0) {
                        cs->pending[ww] = 0;
                        __threadfence_block();
                        cs->ready[ww] = 1;
                    }
                }
                __syncwarp();
                if (lane == 0) atomicExch(&cs->wpoll, 0);
            } else {
                __nanosleep(P.poll_ns);
            }
            if ((spin & 255) == 255) {
                int bad = 0;
                if (lane == 0) {
                    const unsigned long long t = globaltimer();
                    if (t0 == 0) t0 = t;
                    bad = (t - t0 > kWatchdogNs) || *(volatile int *)P.err;
                    if (bad) atomicExch(P.err, 1);
                }
                if (__shfl_sync(0xffffffffu, bad, 0)) return false;
            }
        }
        __syncwarp();
        return true;
    }
    // many distinct requests (wide phases): poll directly
    for (int spin = 0;; ++spin) {
        __nanosleep(P.poll_ns);
        if (*vk >= (unsigned)lvl) break;
        unsigned rem = 0;
        if (has_src) {
            const unsigned cc = ld_relaxed(P.col_done + (size_t)j * kColRep + rep);
            rem = cc >= jneed ? 0u : jneed - cc;
        }
        if (has_own) {
            const unsigned cc = ld_relaxed(P.col_done + (size_t)k * kColRep + rep);
            rem = max(rem, cc >= kneed ? 0u : kneed - cc);
        }
        const unsigned mx = __reduce_max_sync(0xffffffffu, rem);
        if (mx == 0) break;
        if (mx > 4) __nanosleep(min(mx * 32u, 1024u));
        if ((spin & 255) == 255) {
            int bad = 0;
            if (lane == 0) {
                const unsigned long long t = globaltimer();
                if (t0 == 0) t0 = t;
                bad = (t - t0 > kWatchdogNs) || *(volatile int *)P.err;
                if (bad) atomicExch(P.err, 1);
            }
            if (__shfl_sync(0xffffffffu, bad, 0)) return false;
        }
    }
    __syncwarp();
    return true;
}

// kPush item: <= 32 ordered chunks into <= 256 distinct targets of one
// destination column.  Everything static -- the chunk descriptors (one per
// lane), every entry's chunk and target index (u8 map, up to 8 entries per
// lane) and the target offsets -- is loaded before the phase wait; after it,
// ONE round of independent loads fetches the targets, the sources' L
// values, pivots and multipliers.  The targets are staged in shared memory,
// the MACs applied there epoch by epoch (entries of one epoch hit distinct
// targets; only epochs are ordered), and every target written back once.

__device__ __forceinline__ int round_chunk(int rbase, int lane, int nch, int est) {
    const unsigned start_bits = __reduce_or_sync(
        0xffffffffu, (lane < nch && est > rbase && est < rbase + 32) ? (1u << (est - rbase)) : 0u);
    const int cfirst = __popc(__ballot_sync(0xffffffffu, lane < nch && est <= rbase)) - 1;
    return cfirst + __popc(start_bits & ((2u << lane) - 1u));
}

__device__ __forceinline__ void stamp(unsigned long long *rec, int k, int lane) {
    if (rec && lane == 0) rec[k] = globaltimer();
}

template <int KR, int NS>
__device__ __forceinline__ bool run_push(const FactorParams &P, int4 a, int4 b, int4 c, int lane,
                                         CtaSync *cs, double *sg, unsigned long long *rec, int4 na,
                                         int4 nb, int4 nc, int *mycol) {
    const i64 moff = (i64)(unsigned)a.x | ((i64)a.y << 32);
    const i64 toff = (i64)(unsigned)a.z | ((i64)a.w << 32);
    const int base = b.x, c0 = b.y, nch = b.z, ntgt = b.w, macs = c.x;
    const int lvl = c.y >> 2;
    const bool check = *(volatile unsigned *)&cs->known < (unsigned)lvl;
    const int rep = (blockIdx.x + (threadIdx.x >> 5)) % kColRep;
    // own columns: lanes < ncol hold (column, earlier-phase items into it)
    const int ncol = c.w;
    int kcol = -1;
    unsigned kneed = 0, krem = 0, jrem = 0;
    if (lane < ncol) {
        const int2 cd = __ldg(reinterpret_cast<const int2 *>(P.cdeps) + c.z + lane);
        kcol = cd.x;
        kneed = (unsigned)cd.y;
        if (check) {  // first poll of the own-column dependency, in flight early
            const unsigned x = ld_relaxed(P.col_done + (size_t)kcol * kColRep + rep);
            krem = x >= kneed ? 0u : kneed - x;
        }
    }
    *mycol = kcol;
    int4 ch = make_int4(0, 0, 0, 0);
    if (lane < nch) ch = ldp(reinterpret_cast<const int4 *>(P.chunks) + c0 + lane);
    const int cnt = ch.w & 0x7fffffff;
    const bool newep = lane == 0 || (lane < nch && (ch.w & glu::kEpochBit));
    const unsigned epm = __ballot_sync(0xffffffffu, newep);
    const int myep = __popc(epm & ((2u << lane) - 1u)) - 1;
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int x = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += x;
    }
    const int est = incl - cnt;
    const int nr = (macs + 31) >> 5, nt = (ntgt + 31) >> 5;
    int dslot = 0;
    unsigned jneed = 0;
    if (lane < nch) {
        dslot = __ldg(P.diag_pos + ch.y);
        jneed = (unsigned)__ldg(P.col_total + ch.y);
        if (check) {
            const unsigned x = ld_relaxed(P.col_done + (size_t)ch.y * kColRep + rep);
            jrem = x >= jneed ? 0u : jneed - x;
        }
    }
    int u[KR], ci[KR], to[KR];
#pragma unroll
    for (int r = 0; r < KR; ++r) {
        u[r] = -1;
        to[r] = -1;
        if (r < nr) {
            ci[r] = round_chunk(32 * r, lane, nch, est);
            if (32 * r + lane < macs) u[r] = ldp8(P.map8 + moff + 32 * r + lane);
        }
        if (r < nt && 32 * r + lane < ntgt) to[r] = ldp16(P.tgt16 + toff + 32 * r + lane);
    }
    stamp(rec, 3, lane);
    if (__reduce_max_sync(0xffffffffu, max(krem, jrem)) != 0 &&
        !wait_cols(P, lane, lane < nch, ch.y, jneed, lane < ncol, kcol, kneed, lvl, cs, rep))
        return false;
    stamp(rec, 4, lane);
    // value phase: NS value sets per round of loads (batch launches share
    // the static part, the dependency wait and the release across all sets)
    int ep[KR];
#pragma unroll
    for (int r = 0; r < KR; ++r) ep[r] = __shfl_sync(0xffffffffu, myep, r < nr ? ci[r] : 0);
    const int nep = __popc(epm);
    for (int bs0 = 0; bs0 < P.nb; bs0 += NS) {
        double piv[NS], mult[NS], t[NS][KR], l[NS][KR];
#pragma unroll
        for (int ns = 0; ns < NS; ++ns) {
            piv[ns] = 1.0;
            mult[ns] = 0.0;
            if (bs0 + ns >= P.nb) continue;
            const double *V = P.v + (size_t)(bs0 + ns) * P.set_stride;
            if (lane < nch) {
                piv[ns] = ldv(V + dslot);
                mult[ns] = ldv(V + ch.x);
            }
#pragma unroll
            for (int r = 0; r < KR; ++r) {
                if (to[r] >= 0) t[ns][r] = ldv(V + base + to[r]);
                if (r < nr) {
                    const int cp0 = __shfl_sync(0xffffffffu, ch.z, ci[r]);
                    const int cest = __shfl_sync(0xffffffffu, est, ci[r]);
                    if (u[r] >= 0) l[ns][r] = ldv(V + cp0 + (32 * r + lane - cest));
                }
            }
        }
#pragma unroll
        for (int ns = 0; ns < NS; ++ns) {
            if (bs0 + ns >= P.nb) continue;
            double *sgn = sg + ns * (KR * 32);
            double *V = P.v + (size_t)(bs0 + ns) * P.set_stride;
#pragma unroll
            for (int r = 0; r < KR; ++r)
                if (to[r] >= 0) sgn[32 * r + lane] = t[ns][r];
#pragma unroll
            for (int r = 0; r < KR; ++r) {
                if (r < nr) {
                    const double pv = __shfl_sync(0xffffffffu, piv[ns], ci[r]);
                    const double mu = __shfl_sync(0xffffffffu, mult[ns], ci[r]);
                    if (u[r] >= 0) l[ns][r] = __dmul_rn(__ddiv_rn(l[ns][r], pv), mu);  // the product
                }
            }
            __syncwarp();
            if (bs0 + ns == 0) stamp(rec, 5, lane);
            if (nep == 1) {
#pragma unroll
                for (int r = 0; r < KR; ++r)
                    if (u[r] >= 0) sgn[u[r]] = __dsub_rn(sgn[u[r]], l[ns][r]);
            } else {
                for (int e = 0; e < nep; ++e) {
#pragma unroll
                    for (int r = 0; r < KR; ++r)
                        if (u[r] >= 0 && ep[r] == e) sgn[u[r]] = __dsub_rn(sgn[u[r]], l[ns][r]);
                    __syncwarp();
                }
            }
            __syncwarp();
#pragma unroll
            for (int r = 0; r < KR; ++r)
                if (to[r] >= 0) stv(V + base + to[r], sgn[32 * r + lane]);
        }
        __syncwarp();
    }
    __syncwarp();
    stamp(rec, 6, lane);
    return true;
}

// kDeep item: one target, many ordered contributions.  Lanes form 32
// products at a time (independent roundings); every lane then replays the
// subtraction chain in order from shuffles, so the target sees exactly the
// reference's sequence of roundings with one load and one store.  The next
// group's operands are loaded before the current group's chain.
constexpr int kDeepRing = 8;  // deep-ref groups of 32 in flight (cp.async into shared memory)

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem, bool pred) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    const int n = pred ? 16 : 0;  // src-size 0: zero-fill, no global read
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(gmem), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// kDeep item: one target, many ordered contributions.  Lanes form 32
// products at a time (independent roundings); every lane then replays the
// subtraction chain in order from shuffles, so the target sees exactly the
// reference's sequence of roundings with one load and one store.  Two-stage
// pipeline so the serial chain never waits on memory: the {l, d, m} refs
// stream into a shared-memory ring kDeepRing groups ahead (cp.async), the
// three operands of a group are loaded two groups ahead.
__device__ __forceinline__ bool run_deep(const FactorParams &P, int4 a, int4 b, int4 c_, int lane,
                                         CtaSync *cs, int wait_l, int4 *ring, double *sg, int4 na,
                                         int4 nb, int4 nc, unsigned long long *rec) {
    const i64 off = (i64)(unsigned)a.x | ((i64)a.y << 32);
    const int macs = c_.x;
    const int ng = (macs + 31) >> 5;
    const int4 *dr = reinterpret_cast<const int4 *>(P.deep) + off;
    auto issue_ring = [&]() {
#pragma unroll
        for (int g = 0; g < kDeepRing; ++g) {
            cp_async16(ring + g * 32 + lane, dr + min(32 * g + lane, macs - 1), 32 * g + lane < macs);
            cp_async_commit();
        }
    };
    issue_ring();
    if (wait_l >= 0 && !wait_phase(P, wait_l, lane, cs)) {
        cp_async_wait<0>();
        return false;
    }
    stamp(rec, 3, lane);
    // once per value set of the launch (the refs stream again for each)
    for (int bs = 0; bs < P.nb; ++bs) {
    if (bs > 0) issue_ring();
    double *V = P.v + (size_t)bs * P.set_stride;
    double *tp = V + b.x;
    double acc = ldv(tp);
    // operand sets for groups g % 3 (values loaded three groups ahead)
    double l0 = 0.0, d0 = 1.0, m0 = 0.0, l1 = 0.0, d1 = 1.0, m1 = 0.0, l2 = 0.0, d2 = 1.0, m2 = 0.0;
    auto load_group = [&](int grp, double &l, double &d, double &m) {
        if (32 * grp + lane < macs) {
            const int4 r = ring[(grp % kDeepRing) * 32 + lane];
            l = ldv(V + r.x); d = ldv(V + r.y); m = ldv(V + r.z);
        }
    };
    auto refill = [&](int grp) {  // slot of group grp was just consumed: fetch group grp + kDeepRing
        const int gn = grp + kDeepRing;
        cp_async16(ring + (grp % kDeepRing) * 32 + lane, dr + min(32 * gn + lane, macs - 1),
                   32 * gn + lane < macs);
        cp_async_commit();
    };
    cp_async_wait<kDeepRing - 4>();  // groups 0..3 landed
    __syncwarp();
    load_group(0, l0, d0, m0);
    load_group(1, l1, d1, m1);
    load_group(2, l2, d2, m2);
    __syncwarp();
    refill(0); refill(1); refill(2);
    sg[lane] = __dmul_rn(__ddiv_rn(l0, d0), m0);  // products of group 0
    load_group(3, l0, d0, m0);
    __syncwarp();
    refill(3);
    // iteration g: products of group g+1 (set (g+1)%3) -> buffer, reload that
    // set with group g+4, chain group g on lane 0 from shared memory
    auto step = [&](int g, double &l, double &d, double &m) {
        if (g + 1 < ng) sg[((g + 1) & 1) * 32 + lane] = __dmul_rn(__ddiv_rn(l, d), m);
        cp_async_wait<kDeepRing - 1>();  // group g+4 landed
        __syncwarp();
        load_group(g + 4, l, d, m);
        __syncwarp();
        refill(g + 4);
        if (lane == 0) {
            const double2 *pb = reinterpret_cast<const double2 *>(sg + (g & 1) * 32);
            const int cnt = min(32, macs - 32 * g);
            if (cnt == 32) {
#pragma unroll
                for (int s2 = 0; s2 < 16; ++s2) {
                    const double2 x = pb[s2];
                    acc = __dsub_rn(acc, x.x);
                    acc = __dsub_rn(acc, x.y);
                }
            } else {
                for (int s1 = 0; s1 < cnt; ++s1) acc = __dsub_rn(acc, sg[(g & 1) * 32 + s1]);
            }
        }
        __syncwarp();
    };
    for (int g = 0; g < ng; g += 3) {
        step(g, l1, d1, m1);
        if (g + 1 < ng) step(g + 1, l2, d2, m2);
        if (g + 2 < ng) step(g + 2, l0, d0, m0);
    }
    cp_async_wait<0>();
    if (lane == 0) stv(tp, acc);
    __syncwarp();
    }
    stamp(rec, 6, lane);
    if (rec && lane == 0) rec[7] = ng;
    return true;
}

// Pivot check + divide of column j (_kernels.py:152-173): cmax over the
// whole column with the reference's `av > cmax` rule (NaN never wins),
// failure if |piv| <= thresh * cmax, else L(:,j) /= piv.
__device__ __forceinline__ void divide_column(const FactorParams &Pin, int j, int lane, int bs) {
    FactorParams P = Pin;  // value set bs
    P.v = Pin.v + (size_t)bs * Pin.set_stride;
    P.fail = Pin.fail + bs;
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

template <int KR, int NS>
__global__ void __launch_bounds__(kThreads, 1) factor_kernel(FactorParams P) {
    const int lane = threadIdx.x & 31;
    // consecutive items go to consecutive SMs (a thin phase spreads over the chip)
    const int gw = (threadIdx.x >> 5) * gridDim.x + blockIdx.x;
    const int nw = gridDim.x * kWarps;
    __shared__ __align__(16) double stage[kWarps * glu::kMaxItemMacs];
    __shared__ CtaSync cs;
    double *sg = stage + (threadIdx.x >> 5) * glu::kMaxItemMacs;
    if (threadIdx.x == 0) {
        cs.known = 0;
        cs.polling = 0;
        cs.wpoll = 0;
    }
    if (threadIdx.x < kWarps) {
        cs.pending[threadIdx.x] = 0;
        cs.ready[threadIdx.x] = 0;
    }
    __syncthreads();
    if (P.level_ns && blockIdx.x == 0 && threadIdx.x == 0) P.level_ns[0] = globaltimer();
    // this warp's items: consecutive items on consecutive SMs
    const int q_hi = P.n_items, g0 = gw, qstride = nw;
    int cur = -1, coarse = 0, nq = 0;
    unsigned ran = 0;
    __shared__ WarpQ wqs[kWarps];
    extern __shared__ int4 rings[];  // kWarps * kDeepRing * 32 (dynamic: > 48 KB static limit)
    WarpQ *wq = wqs + (threadIdx.x >> 5);
    int4 *ring = rings + (threadIdx.x >> 5) * kDeepRing * 32;
    int4 a = make_int4(0, 0, 0, 0), b = a, c = a;
    if (g0 < q_hi) {
        const int4 *ip = reinterpret_cast<const int4 *>(P.items + g0);
        a = ldp(ip); b = ldp(ip + 1); c = ldp(ip + 2);
    }
    for (int it = g0; it < q_hi; it += qstride) {
        // next item's descriptor in flight while this one runs
        const int nit = it + qstride;
        int4 na = a, nb = b, nc = make_int4(0, -4, 0, 0);
        if (nit < q_hi) {
            const int4 *ip = reinterpret_cast<const int4 *>(P.items + nit);
            na = ldp(ip); nb = ldp(ip + 1); nc = ldp(ip + 2);
        }
        // (nc.y = -4 when there is no next item: a phase end)
        const int lvl = c.y >> 2;
        if (lvl != cur) {
            ran = 0;
            cur = lvl;
        }
        // deep items wait for every earlier phase (coarse), once per phase
        int wait_l = -1;
        if ((c.y & 1) && coarse < lvl) {
            wait_l = lvl - 1;
            coarse = lvl;
        }
        unsigned long long *rec = nullptr;
        if (P.trace && it >= P.trace_i0 && it < P.trace_i1) {
            rec = P.trace + 8 * (size_t)(it - P.trace_i0);
            if (lane == 0) {
                rec[0] = (unsigned long long)it | ((unsigned long long)lvl << 32);
                rec[1] = gw;
                rec[2] = globaltimer();
            }
        }
        int mycol = -1;  // lanes < ncol: the item's destination columns
        bool ok;
        if (c.y & 1) {
            if (lane == 0) mycol = __ldg(reinterpret_cast<const int2 *>(P.cdeps) + c.z).x;
            ok = run_deep(P, a, b, c, lane, &cs, wait_l, ring, sg, na, nb, nc, rec);
        } else {
            ok = run_push<KR, NS>(P, a, b, c, lane, &cs, sg, rec, na, nb, nc, &mycol);
        }
        if (!ok) return;
        ++ran;
        finish_item(P, wq, nq, mycol, (c.y & 1) ? 1 : c.w, (c.y >> 1) & 1, lvl, ran,
                    (nc.y >> 2) != lvl, lane);
        if (rec && lane == 0 && !(c.y & 1)) rec[7] = globaltimer() | (1ull << 63);
        a = na; b = nb; c = nc;
    }
    // every phase complete -> pivot check + divide of every column
    if (P.n_levels > 0 && !wait_phase(P, P.n_levels - 1, lane, &cs)) return;
    for (int bs = 0; bs < P.nb; ++bs)
        for (int j = gw; j < P.n_div; j += nw) divide_column(P, j, lane, bs);
}

// ---------------------------------------------------------------------------
// Dense tail: one thread-block cluster factors the trailing m x m block
// (columns t0..n-1, each alone in one of the last m phases) in distributed
// shared memory, as a blocked right-looking LU with panels of b columns.
// CTA c of C owns panels c, c+C, ... (all m tail rows of their columns,
// dense, plus a structure bitmask).  For panel p (sources s0..s1-1):
//   * the owner of panel p+1 first applies panel p to it, factors it
//     (source by source, __syncthreads between sources) and publishes its
//     divided L columns and structure to a double-buffered global slot
//     (lookahead: the critical path never waits for trailing updates);
//   * every CTA applies panel p to its later columns: the panel rows of a
//     column first (a b x b triangular sweep, one warp per column), then
//     every row below the panel with the target held in a register across
//     the b sources;
//   * one cluster barrier per panel.
// Per target the MACs are the reference's: A(i,q) -= (A(i,s) / A(s,s)) *
// A(s,q), three roundings, ascending source s (= ascending phase here), and
// only where L(i,s) and U(s,q) are in the pattern -- bitwise identical to
// the sparse path for both contracts.  Finally every CTA writes its columns
// back (undivided) and pivot-checks/divides them.
// ---------------------------------------------------------------------------
namespace cg = cooperative_groups;
constexpr int kTailThreads = 512;
constexpr int kTailB = 16;  // largest panel width (register arrays)
constexpr int kTailMaxLocal = 256;  // owned columns per CTA

struct TailParams {
    double *v;
    const i32 *col_ptr, *row_idx, *diag_pos, *level_of;
    i32 t0, m, mpad, mw, b, np, ncl;
    i32 gstride;  // doubles per panel slot: b x mpad divided L values, then mpad u32 row words
                  // (bit k of row i: L(i, s0 + k) in the pattern)
    double *G;    // one slot per panel
    unsigned *ready;  // per panel: published (zeroed before each launch)
    double thresh;
    unsigned long long *fail;
    i32 fail_by_column;
    const unsigned long long *mk0;  // structure bitmasks of the tail columns (m x mw, host-built)
    const i32 *blk;     // per tail column: first slot inside the block (rows >= t0)
    double *umax;       // per tail column: max |value| above the block (final before the tail)
    // batched launches: cluster b factors value set b (its own values,
    // panel slots, ready flags, failure key and maxima)
    long long set_stride, g_set;
    // diagnostics (option 13): [0..7] CTA 0 phase stamps, then per panel
    // {observed p-1, applied p-1 to it, column sweep done, written back, published} by its owner
    unsigned long long *trace;
};

__device__ __forceinline__ bool mbit(const unsigned long long *mk, int i) {
    return (mk[i >> 6] >> (i & 63)) & 1ull;
}
// bits [s, s+len) of a row mask, len <= 16
__device__ __forceinline__ unsigned mbits(const unsigned long long *mk, int s, int len) {
    const int w = s >> 6, o = s & 63;
    unsigned long long x = mk[w] >> o;
    if (o + len > 64) x |= mk[w + 1] << (64 - o);
    return (unsigned)(x & ((1ull << len) - 1ull));
}


__global__ void __launch_bounds__(kTailThreads, 1) tail_kernel(TailParams T0) {
    TailParams T = T0;
    {
        const int set = (int)(blockIdx.x / cg::this_cluster().num_blocks());
        T.v += (size_t)set * T.set_stride;
        T.G += (size_t)set * T.g_set;
        T.ready = reinterpret_cast<unsigned *>(T.G + (size_t)T.np * T.gstride);
        T.fail += set;
        T.umax += (size_t)set * T.m;
        if (set > 0) T.trace = nullptr;
    }
    extern __shared__ __align__(16) double tsm[];
    __shared__ double tri[kTailB * kTailB];   // panel rows' divided L values (row-major [i][s])
    __shared__ unsigned tribits[kTailB];      // L structure of panel row i over the panel sources
    __shared__ int qtab[kTailMaxLocal];       // local column -> tail column (M: none)
    __shared__ double urow[2][kTailB];        // factor_panel: U(s, panel) broadcast
    __shared__ unsigned ubits[2];
    // the cluster guarantees the C CTAs are co-resident (the panel flags rely on it)
    cg::cluster_group cl = cg::this_cluster();
    const int C = (int)cl.num_blocks(), c = (int)cl.block_rank();
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5, nwarp = nt >> 5;
    const int B = T.b, M = T.m;
    double *cols = tsm;
    unsigned long long *mk = reinterpret_cast<unsigned long long *>(tsm + (size_t)T.ncl * T.mpad);
    const int npl = c < T.np ? (T.np - c + C - 1) / C : 0;  // owned panels
    const int ncol = min(npl * B, T.ncl);
    // owned column q -> local index (owner = (q / B) % C); the divisions run
    // once here, the loops read the table
    auto xloc = [&](int q) { return ((q / B) / C) * B + (q % B); };
    for (int x = tid; x < kTailMaxLocal; x += nt) {
        const int q = x < ncol ? ((x / B) * C + c) * B + (x % B) : M;
        qtab[x] = q < M ? q : M;
    }
    __syncthreads();
    auto qglob = [&](int x) { return qtab[x]; };
    auto stamp_t = [&](int k) {
        if (T.trace && tid == 0) T.trace[k] = globaltimer();
    };
    if (c == 0) stamp_t(0);
    int nvalid = ncol;  // owned columns that exist (the last panel may be short)
    while (nvalid > 0 && qtab[nvalid - 1] >= M) --nvalid;
    // load the owned columns: zero-fill, structure masks from the host-built
    // table, then a warp per column with its entry loads batched
    for (int e = tid; e < nvalid * T.mpad; e += nt) cols[e] = 0.0;
    for (int e = tid; e < nvalid * T.mw; e += nt) {
        const int x = e / T.mw;
        mk[e] = __ldg(T.mk0 + (size_t)qglob(x) * T.mw + (e - x * T.mw));
    }
    __syncthreads();
    for (int x = wid; x < nvalid; x += nwarp) {
        const int j = T.t0 + qglob(x);
        const int lo = __ldg(T.blk + qglob(x)), hi = __ldg(T.col_ptr + j + 1);  // block rows only
        double *cq = cols + (size_t)x * T.mpad;
#pragma unroll 4
        for (int p = lo + lane; p < hi; p += 32) {
            const int r = __ldg(T.row_idx + p) - T.t0;
            const double val = ldv(T.v + p);
            if (r >= 0) cq[r] = val;
        }
    }
    __syncthreads();
    if (c == 0) stamp_t(1);
    // Column maxima above the block (the U rows: final before this kernel),
    // for the pivot test at the end.  Work units of <= 1024 entries are dealt
    // over the warps (the power/ground hub columns hold ~34k each); the
    // apply phase's tri[] array accumulates the bits of the non-negative
    // maxima.  NaN never wins, as in the reference's `av > cmax`.
    auto umax_pass = [&]() {
        unsigned long long *acc = reinterpret_cast<unsigned long long *>(tri);
        for (int x = tid; x < kTailMaxLocal; x += nt) acc[x] = 0ull;
        __syncthreads();
        int u = 0;
        for (int x = 0; x < nvalid; ++x) {
            const int j = T.t0 + qglob(x);
            const int lo = __ldg(T.col_ptr + j), hb = __ldg(T.blk + qglob(x));
            for (int p0 = lo; p0 < hb; p0 += 1024, ++u) {
                if (u % nwarp != wid) continue;
                const int p1 = min(p0 + 1024, hb);
                double m = 0.0;
#pragma unroll 8
                for (int p = p0 + lane; p < p1; p += 32) {
                    const double av = fabs(ldv(T.v + p));
                    if (av > m) m = av;
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const double y = __shfl_xor_sync(0xffffffffu, m, o);
                    if (y > m) m = y;
                }
                if (lane == 0 && m > 0.0) atomicMax(acc + x, (unsigned long long)__double_as_longlong(m));
            }
        }
        __syncthreads();
        for (int x = tid; x < nvalid; x += nt) T.umax[qglob(x)] = __longlong_as_double((long long)acc[x]);
        __syncthreads();
    };
    // CTAs 0 and 1 own the first panels (needed before a pass of ~30 us
    // would end): they run it at the end, where they have slack
    if (c >= 2) umax_pass();
    const int ia = tid, ib = tid + nt;  // this thread's rows (m <= 2 * nt)

    // Owner: factor panel pp in place (its columns already hold every update
    // from earlier panels) and publish the divided L columns + structure.
    // The panel lives in registers while it is factored: each thread holds
    // its rows of the b panel columns; per source one __syncthreads, through
    // which the owner of row s broadcasts U(s, panel) and its structure.
    auto factor_panel = [&](int pp) {
        const int s0 = pp * B, s1 = min(s0 + B, M), bp = s1 - s0;
        const int xb0 = xloc(s0);  // the panel's columns are consecutive local columns
        double *g = T.G + (size_t)pp * T.gstride;
        unsigned *grow = reinterpret_cast<unsigned *>(g + (size_t)B * T.mpad);
        double ra[kTailB], rb[kTailB];
        unsigned pa = 0, pb = 0;  // bit k: row ia / ib is in panel column s0+k
        // warps whose rows all lie above the panel (or past M) have nothing
        // to update in it: their chains would only subtract +0.0 (the sweep
        // is FP64-bound on the owner SM, so they are skipped -- measured
        // ~550 + 70 x (remaining columns) cycles per step with them)
        const bool wa = __any_sync(0xffffffffu, ia < M && ia >= s0);
        const bool wb = __any_sync(0xffffffffu, ib < M && ib >= s0);
#pragma unroll
        for (int k = 0; k < kTailB; ++k) {
            ra[k] = 0.0;
            rb[k] = 0.0;
            if (k < bp) {
                const double *cq = cols + (size_t)(xb0 + k) * T.mpad;
                const unsigned long long *mq = mk + (xb0 + k) * T.mw;
                if (ia < M) { ra[k] = cq[ia]; pa |= (unsigned)mbit(mq, ia) << k; }
                if (ib < M) { rb[k] = cq[ib]; pb |= (unsigned)mbit(mq, ib) << k; }
            }
        }
        unsigned bra = 0, brb = 0;
#pragma unroll
        for (int k = 0; k < kTailB; ++k) {
            if (k < bp) {
                const int s = s0 + k;
                double *ur = urow[k & 1];
                if (ia == s) {
#pragma unroll
                    for (int kk = 0; kk < kTailB; ++kk) ur[kk] = ra[kk];
                    ubits[k & 1] = pa;
                }
                if (ib == s) {
#pragma unroll
                    for (int kk = 0; kk < kTailB; ++kk) ur[kk] = rb[kk];
                    ubits[k & 1] = pb;
                }
                __syncthreads();
                const double piv = ur[k];
                const unsigned ub = ubits[k & 1];
                const bool ba = ia > s && ia < M && ((pa >> k) & 1u);
                const bool bb = ib > s && ib < M && ((pb >> k) & 1u);
                double la = 0.0, lb = 0.0;
                if (ba) { la = __ddiv_rn(ra[k], piv); __stcg(g + (size_t)k * T.mpad + ia, la); bra |= 1u << k; }
                if (bb) { lb = __ddiv_rn(rb[k], piv); __stcg(g + (size_t)k * T.mpad + ib, lb); brb |= 1u << k; }
                // branch-free: every product is formed, the subtraction is
                // selected only where L(i,s) and U(s,q) are in the pattern
                const unsigned ma = ba ? ub : 0u, mb = bb ? ub : 0u;
                if (wa) {
#pragma unroll
                    for (int kk = k + 1; kk < kTailB; ++kk)
                        ra[kk] = __dsub_rn(ra[kk], ((ma >> kk) & 1u) ? __dmul_rn(la, ur[kk]) : 0.0);
                }
                if (wb) {
#pragma unroll
                    for (int kk = k + 1; kk < kTailB; ++kk)
                        rb[kk] = __dsub_rn(rb[kk], ((mb >> kk) & 1u) ? __dmul_rn(lb, ur[kk]) : 0.0);
                }
            }
        }
        stamp_t(8 + 6 * pp + 2);
#pragma unroll
        for (int k = 0; k < kTailB; ++k) {
            if (k < bp) {
                double *cq = cols + (size_t)(xb0 + k) * T.mpad;
                if (wa && ia < M) cq[ia] = ra[k];
                if (wb && ib < M) cq[ib] = rb[k];
            }
        }
        if (ia < M) __stcg(grow + ia, bra);
        if (ib < M) __stcg(grow + ib, brb);
        __syncthreads();
    };

    // Apply panel p to the owned columns with local index in [xa, xb) that lie
    // beyond the panel.
    auto apply_panel = [&](int p, int xa, int xb) {
        const int s0 = p * B, s1 = min(s0 + B, M), bp = s1 - s0;
        const double *g = T.G + (size_t)p * T.gstride;
        const unsigned *grow = reinterpret_cast<const unsigned *>(g + (size_t)B * T.mpad);
        // the b x b triangle of divided L values among the panel rows (loads
        // are unconditional: entries outside the pattern are never used)
        for (int e = tid; e < kTailB * kTailB; e += nt) {
            const int i = e / kTailB, k = e % kTailB;  // panel row s0+i, source s0+k
            tri[e] = (i < bp && k < i) ? __ldcg(g + (size_t)k * T.mpad + s0 + i) : 0.0;
        }
        if (tid < kTailB) tribits[tid] = tid < bp ? __ldcg(grow + s0 + tid) : 0u;
        // this thread's rows below the panel: structure word + divided L values
        double la[kTailB], lb[kTailB];
        const unsigned bitsa = (ia >= s1 && ia < M) ? __ldcg(grow + ia) : 0u;
        const unsigned bitsb = (ib >= s1 && ib < M) ? __ldcg(grow + ib) : 0u;
        // only rows below the panel use its L values (bitsa/bitsb are 0 above)
        const bool ra = ia >= s1 && ia < M, rb = ib >= s1 && ib < M;
#pragma unroll
        for (int k = 0; k < kTailB; ++k) {
            la[k] = (ra && k < bp) ? __ldcg(g + (size_t)k * T.mpad + ia) : 0.0;
            lb[k] = (rb && k < bp) ? __ldcg(g + (size_t)k * T.mpad + ib) : 0.0;
        }
        __syncthreads();
        // (A) panel rows of each column: a warp per column, lane = panel row
        for (int x = xa + wid; x < xb; x += nwarp) {
            if (qglob(x) < s1) continue;
            double *cq = cols + (size_t)x * T.mpad;
            const unsigned ub = mbits(mk + x * T.mw, s0, bp);
            const unsigned lbits = lane < bp ? tribits[lane] : 0u;
            for (int k = 0; k + 1 < bp; ++k) {
                const double mult = cq[s0 + k];
                if (((ub >> k) & 1u) && lane > k && lane < bp && ((lbits >> k) & 1u))
                    cq[s0 + lane] = __dsub_rn(cq[s0 + lane], __dmul_rn(tri[lane * kTailB + k], mult));
                __syncwarp();
            }
        }
        __syncthreads();
        // (B) rows below the panel, target in a register across the b sources;
        // two columns at a time so each thread carries independent chains
        int x = xa;
        xb = min(xb, nvalid);
        while (x < xb && qglob(x) < s1) ++x;  // owned columns beyond the panel are contiguous
        for (; x + 1 < xb; x += 2) {
            double *c0 = cols + (size_t)x * T.mpad, *c1 = cols + (size_t)(x + 1) * T.mpad;
            const unsigned u0 = mbits(mk + x * T.mw, s0, bp), u1 = mbits(mk + (x + 1) * T.mw, s0, bp);
            const unsigned a0 = u0 & bitsa, a1 = u1 & bitsa, b0 = u0 & bitsb, b1 = u1 & bitsb;
            if (a0 | a1) {
                double t0 = c0[ia], t1 = c1[ia];
#pragma unroll
                for (int k = 0; k < kTailB; ++k) {
                    // absent MACs contribute +0.0 (an exact no-op): no select in the chain
                    t0 = __dsub_rn(t0, ((a0 >> k) & 1u) ? __dmul_rn(la[k], c0[s0 + k]) : 0.0);
                    t1 = __dsub_rn(t1, ((a1 >> k) & 1u) ? __dmul_rn(la[k], c1[s0 + k]) : 0.0);
                }
                c0[ia] = t0;
                c1[ia] = t1;
            }
            if (b0 | b1) {
                double t0 = c0[ib], t1 = c1[ib];
#pragma unroll
                for (int k = 0; k < kTailB; ++k) {
                    t0 = __dsub_rn(t0, ((b0 >> k) & 1u) ? __dmul_rn(lb[k], c0[s0 + k]) : 0.0);
                    t1 = __dsub_rn(t1, ((b1 >> k) & 1u) ? __dmul_rn(lb[k], c1[s0 + k]) : 0.0);
                }
                c0[ib] = t0;
                c1[ib] = t1;
            }
        }
        for (; x < xb; ++x) {
            double *cq = cols + (size_t)x * T.mpad;
            const unsigned ub = mbits(mk + x * T.mw, s0, bp);
            const unsigned ua = ub & bitsa, ubb = ub & bitsb;
            if (ua) {
                double t = cq[ia];
#pragma unroll
                for (int k = 0; k < kTailB; ++k)
                    t = __dsub_rn(t, ((ua >> k) & 1u) ? __dmul_rn(la[k], cq[s0 + k]) : 0.0);
                cq[ia] = t;
            }
            if (ubb) {
                double t = cq[ib];
#pragma unroll
                for (int k = 0; k < kTailB; ++k)
                    t = __dsub_rn(t, ((ubb >> k) & 1u) ? __dmul_rn(lb[k], cq[s0 + k]) : 0.0);
                cq[ib] = t;
            }
        }
        __syncthreads();
    };

    // Panel p is published once (its own G slot) with a release flag; a CTA
    // waits only for the flag of the panel it applies next -- no cluster-wide
    // barrier, so nobody waits for another CTA's trailing updates.
    auto publish = [&](int pp) {
        __syncthreads();
        if (tid == 0) {
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
            asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(T.ready + pp), "r"(1u) : "memory");
        }
    };
    auto await = [&](int pp) {
        if (tid == 0) {
            unsigned f;
            do {
                asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(T.ready + pp) : "memory");
            } while (f == 0);
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
        }
        __syncthreads();
    };
    const int qmax = nvalid > 0 ? qtab[nvalid - 1] : -1;  // no panel beyond it concerns this CTA
    if (T.np > 0 && c == 0) {
        stamp_t(8 + 1);  // panel 0: observed = applied
        factor_panel(0);
        stamp_t(8 + 3);
        publish(0);
        stamp_t(8 + 4);
    }
    for (int p = 0; p < T.np; ++p) {
        if (p * B > qmax) break;  // no owned column beyond this panel
        await(p);
        const int pn = p + 1;
        const bool own_next = pn < T.np && (pn % C) == c;
        if (own_next) {  // lookahead: the next panel first
            stamp_t(8 + 6 * pn);
            const int xn = xloc(pn * B);
            apply_panel(p, xn, min(xn + B, ncol));
            stamp_t(8 + 6 * pn + 1);
            factor_panel(pn);
            stamp_t(8 + 6 * pn + 3);
            publish(pn);
            stamp_t(8 + 6 * pn + 4);
            const int xl = xn + B;
            apply_panel(p, 0, xn);
            apply_panel(p, xl, ncol);
        } else {
            apply_panel(p, 0, ncol);
        }
    }
    if (c == 0) stamp_t(2);
    if (c < 2) umax_pass();
    // store + pivot check + divide, a warp per column: the column maximum is
    // the one above the block (umax) and the block's own (a scan of the
    // column in shared memory: absent rows hold zeros), as divide_columns
    // takes it over the whole column (_kernels.py:152-173)
    for (int x = wid; x < nvalid; x += nwarp) {
        const int q = qglob(x), j = T.t0 + q;
        const int hb = __ldg(T.blk + q), hi = __ldg(T.col_ptr + j + 1);
        const int d = __ldg(T.diag_pos + j);
        const double *cq = cols + (size_t)x * T.mpad;
        double cmax = __ldcg(T.umax + q);
        for (int r = lane; r < M; r += 32) {
            const double av = fabs(cq[r]);
            if (av > cmax) cmax = av;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double y = __shfl_xor_sync(0xffffffffu, cmax, o);
            if (y > cmax) cmax = y;
        }
        const double piv = cq[q];
        const bool bad = fabs(piv) <= __dmul_rn(T.thresh, cmax);
        if (bad && lane == 0) {
            const unsigned long long key =
                T.fail_by_column ? (unsigned long long)j
                                 : (((unsigned long long)__ldg(T.level_of + j)) << 32) | (unsigned)j;
            atomicMin(T.fail, key);
        }
#pragma unroll 4
        for (int p = hb + lane; p < hi; p += 32) {
            const double val = cq[__ldg(T.row_idx + p) - T.t0];
            stv(T.v + p, (!bad && p > d) ? __ddiv_rn(val, piv) : val);
        }
    }
    __syncthreads();
    if (c == 0) stamp_t(4);
}

struct TailShape;
int tail_gstride(const TailShape &t);
struct TailShape {
    int C = 0, b = 0, np = 0;
    size_t smem = 0;
    int mpad = 0, mw = 0, ncl = 0;
};

int tail_gstride(const TailShape &t) {
    return (int)((((size_t)t.b * t.mpad + (size_t)t.mpad / 2 + 1) + 31) & ~(size_t)31);
}
// one value set's tail scratch: np panel slots, then np ready flags (+ pad)
constexpr int kMaxTailSets = 16;  // = kMaxBatchPerLaunch
long long tail_set_doubles(const TailShape &t) {
    return (long long)t.np * tail_gstride(t) + ((long long)t.np + 32 + 1) / 2 + 16;
}

TailShape tail_shape(int m, int C, int b) {
    TailShape t;
    t.C = C;
    t.b = b;
    t.mpad = (m + 1) & ~1;
    t.mw = (m + 63) / 64;
    t.np = (m + b - 1) / b;
    t.ncl = ((t.np + C - 1) / C) * b;
    t.smem = (size_t)t.ncl * t.mpad * sizeof(double) + (size_t)t.ncl * t.mw * sizeof(unsigned long long);
    return t;
}

// Largest launchable cluster whose shared memory holds an m-column tail, with
// the widest panel that fits (m <= 0: report the capacity only).
TailShape pick_tail(int m, int *cap_out) {
    int dev = 0, optin = 0;
    TailShape best;
    if (cap_out) *cap_out = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
        return best;
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, (const void *)tail_kernel) != cudaSuccess) return best;
    const size_t budget = (size_t)optin - fa.sharedSizeBytes;  // dynamic = opt-in limit - static
    cudaFuncSetAttribute((const void *)tail_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute((const void *)tail_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)budget);
    for (int C : {16, 8, 4, 2}) {
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = C;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(C);
        cfg.blockDim = dim3(kTailThreads);
        cfg.dynamicSmemBytes = budget;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int nclusters = 0;
        if (cudaOccupancyMaxActiveClusters(&nclusters, (const void *)tail_kernel, &cfg) != cudaSuccess ||
            nclusters < 1) {
            cudaGetLastError();
            continue;
        }
        int cap = 0;
        auto fits = [&](int mm, int bb) {
            const TailShape t = tail_shape(mm, C, bb);
            return t.smem <= budget && t.ncl <= kTailMaxLocal;
        };
        while (cap + 1 <= 2 * kTailThreads && fits(cap + 1, 4)) ++cap;
        if (cap_out && cap > *cap_out) *cap_out = cap;
        int bmax = 16;  // widest panel that fits (GLU_TAIL_B caps it: tuning)
        if (const char *e = std::getenv("GLU_TAIL_B")) bmax = std::max(4, std::min(16, std::atoi(e)));
        if (m > 0)
            for (int b : {16, 8, 4})
                if (b <= bmax && fits(m, b)) return tail_shape(m, C, b);
    }
    return best;
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
constexpr int kSolveRing = 4;  // entry-index chunks in flight per warp (cp.async)

__device__ __forceinline__ void cp_async4(void *smem, const void *gmem, bool pred) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    const int n = pred ? 4 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(sa), "l"(gmem), "r"(n) : "memory");
}


// ---------------------------------------------------------------------------
// Dataflow triangular solves (default): no grid barrier.  Every unknown of
// the solve's OUTPUT vector holds a signalling-NaN sentinel until its row is
// done; IEEE arithmetic never produces a signalling NaN, so one relaxed
// 8-byte load both observes "ready" and fetches the value -- no flags, no
// fences.  Rows are taken in level order from a ticket counter, so a row
// waits only on rows with smaller tickets, all held by running warps
// (cooperative launch): deadlock-free.  A long row streams its chain chunk
// by chunk as its inputs arrive instead of waiting for its level.
//
// Buffers: the L pass reads b from X, writes y to Y (all-sentinel on entry)
// and leaves X all-sentinel; the U pass reads y from Y, restores Y to the
// sentinel and writes x to X.  Between calls Y is all-sentinel.
// ---------------------------------------------------------------------------
constexpr unsigned long long kSent = 0x7FF4DEAD5EB17A11ull;  // signalling NaN
constexpr unsigned long long kQuietBit = 1ull << 51;

struct SolveDfParams {
    const double *v;
    long long v_stride;   // batch solves: right-hand side r uses factors v + r * v_stride
    const double *in;     // L: b (X), U: y (Y)
    double *out;          // L: y (Y), U: x (X)
    double *reset;        // L: X (set to sentinel), U: Y (restored to sentinel)
    long long ld_in, ld_out, ld_reset;
    const i32 *rows;      // level-sorted
    const i32 *ent_ptr, *ent_col, *ent_slot;
    const i32 *diag_pos;
    i32 n;
    i32 upper;
    i32 nrhs;
    i32 tblock;           // tasks per ticket grab; 0 = static round-robin over the warps
    i32 in_il, reset_il;  // multi-RHS kernel: in / reset interleaved (out always is)
    // single-RHS dense-tail mode: CTA 0 solves the tail rows [tail_t0, n) in
    // index order with their values also in its shared memory; the other
    // CTAs take the rows_nt list (the rest, level order) by ticket
    i32 tail_t0, n_tail, n_nt;
    const i32 *rows_nt;   // L: followed by the tail rows' partial tasks (n_nt + n_tail tickets)
    const i32 *lsplit;    // L tail row k: first entry in a tail column
    double *part;         // L tail row k: partial sum over the columns left of the block (sentinel)
    unsigned int *ticket;
    unsigned int *err;
};

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const double *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u64(double *p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

constexpr int kSolveTailMax = 1024;  // dense-tail rows CTA 0 keeps in shared memory

__device__ __forceinline__ unsigned long long ld_volatile_smem_u64(const unsigned long long *p) {
    return *reinterpret_cast<const volatile unsigned long long *>(p);
}

__global__ void __launch_bounds__(kThreads, 1) solve_df_kernel(SolveDfParams S) {
    __shared__ __align__(16) double pbuf[kWarps][32];
    __shared__ int icol[kWarps][kSolveRing][32], islot[kWarps][kSolveRing][32];
    __shared__ unsigned long long ysm[kSolveTailMax];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const bool tail_on = S.n_tail > 0;
    // one row of one right-hand side; tail: tail columns read from ysm
    // mode 0: a whole row; 1: a tail row on CTA 0 (tail columns from ysm;
    // in L it starts from its partial sum); 2: an L tail row's partial sum
    // over the columns left of the block (published to S.part)
    auto row = [&](int i, int r, int mode) -> bool {
        const bool tail = mode == 1;
        const double *Xin = S.out + (size_t)r * S.ld_out;  // rows read by this row (ready-or-sentinel)
        const double *V = S.v + (size_t)r * S.v_stride;    // this task's factors
        auto ldx = [&](int c) -> unsigned long long {
            return (tail && c >= S.tail_t0) ? ld_volatile_smem_u64(ysm + (c - S.tail_t0))
                                            : ld_relaxed_u64(Xin + c);
        };
        int e0 = __ldg(S.ent_ptr + i), e1 = __ldg(S.ent_ptr + i + 1);
        double acc;
        if (mode == 2) {
            e1 = __ldg(S.lsplit + (i - S.tail_t0));
            acc = ldv(S.in + (size_t)r * S.ld_in + i);
        } else if (tail && !S.upper) {  // continue from the partial sum
            e0 = __ldg(S.lsplit + (i - S.tail_t0));
            double *pp = S.part + (i - S.tail_t0);
            unsigned long long pb = 0;
            const unsigned long long t0 = globaltimer();
            if (lane == 0) {
                while ((pb = ld_relaxed_u64(pp)) == kSent) {
                    if (globaltimer() - t0 > kWatchdogNs) { atomicExch(S.err, 1u); break; }
                }
                st_relaxed_u64(pp, kSent);  // the buffer returns to the sentinel
            }
            pb = __shfl_sync(0xffffffffu, pb, 0);
            if (pb == kSent) return false;  // watchdog (warp-uniform)
            acc = __longlong_as_double((long long)pb);
        } else {
            acc = ldv(S.in + (size_t)r * S.ld_in + i);
        }
        const int ne = e1 - e0, ng = (ne + 31) >> 5;
        auto ent = [&](int k) { return S.upper ? (e1 - 1 - k) : (e0 + k); };
        auto issue_idx = [&](int g) {
            const int k = 32 * g + lane;
            const int e = ent(min(k, ne - 1));
            cp_async4(&icol[w][g % kSolveRing][lane], S.ent_col + e, k < ne);
            cp_async4(&islot[w][g % kSolveRing][lane], S.ent_slot + e, k < ne);
            cp_async_commit();
        };
        if (ne > 0) {
#pragma unroll
            for (int g = 0; g < kSolveRing; ++g) issue_idx(g);
            unsigned long long xa = 0;
            double va = 0.0;
            cp_async_wait<kSolveRing - 1>();
            __syncwarp();
            if (lane < ne) {
                xa = ldx(icol[w][0][lane]);
                va = ldv(V + islot[w][0][lane]);
            }
            for (int g = 0; g < ng; ++g) {
                unsigned long long xb = 0;
                double vb = 0.0;
                cp_async_wait<kSolveRing - 2>();
                __syncwarp();
                const bool live = 32 * g + lane < ne;
                // chunk g's inputs: re-poll the lanes whose row is not done yet
                if (__any_sync(0xffffffffu, live && xa == kSent)) {
                    const unsigned long long t0 = globaltimer();
                    const int c = icol[w][g % kSolveRing][lane];
                    while (true) {
                        const bool pend = live && xa == kSent;
                        if (!__any_sync(0xffffffffu, pend)) break;
                        if (pend) xa = ldx(c);
                        if (__shfl_sync(0xffffffffu, globaltimer() - t0 > kWatchdogNs, 0)) {
                            if (lane == 0) atomicExch(S.err, 1u);
                            return false;  // warp-uniform
                        }
                    }
                }
                if (32 * (g + 1) + lane < ne) {
                    xb = ldx(icol[w][(g + 1) % kSolveRing][lane]);
                    vb = ldv(V + islot[w][(g + 1) % kSolveRing][lane]);
                }
                __syncwarp();
                issue_idx(g + kSolveRing);
                const double x = __longlong_as_double((long long)xa);
                const bool use = live && (S.upper ? true : (x != 0.0));
                pbuf[w][lane] = use ? __dmul_rn(va, x) : 0.0;
                __syncwarp();
                if (lane == 0) {
                    const double2 *pb = reinterpret_cast<const double2 *>(pbuf[w]);
                    const int cnt = min(32, ne - 32 * g);
                    if (cnt == 32) {
#pragma unroll
                        for (int s2 = 0; s2 < 16; ++s2) {
                            const double2 p2 = pb[s2];
                            acc = __dsub_rn(acc, p2.x);
                            acc = __dsub_rn(acc, p2.y);
                        }
                    } else {
                        for (int s1 = 0; s1 < cnt; ++s1) acc = __dsub_rn(acc, pbuf[w][s1]);
                    }
                }
                __syncwarp();
                xa = xb;
                va = vb;
            }
            cp_async_wait<0>();
            __syncwarp();
        }
        if (lane == 0 && mode == 2) {
            unsigned long long bits = (unsigned long long)__double_as_longlong(acc);
            if (bits == kSent) bits |= kQuietBit;
            st_relaxed_u64(S.part + (i - S.tail_t0), bits);
        } else if (lane == 0) {
            if (S.upper) acc = __ddiv_rn(acc, ldv(V + __ldg(S.diag_pos + i)));
            unsigned long long bits = (unsigned long long)__double_as_longlong(acc);
            if (bits == kSent) bits |= kQuietBit;  // only an untouched input can carry it
            st_relaxed_u64(S.out + (size_t)r * S.ld_out + i, bits);
            st_relaxed_u64(S.reset + (size_t)r * S.ld_reset + i, kSent);
            if (tail) *reinterpret_cast<volatile unsigned long long *>(ysm + (i - S.tail_t0)) = bits;
        }
        __syncwarp();
        return true;
    };
    if (tail_on && blockIdx.x == 0) {
        // the dense tail: rows in index order (a topological order of both
        // passes), a warp per row, hand-offs through shared memory
        for (int k = threadIdx.x; k < S.n_tail; k += blockDim.x) ysm[k] = kSent;
        __syncthreads();
        for (int k = w; k < S.n_tail; k += kWarps) {
            const int i = S.upper ? (S.tail_t0 + S.n_tail - 1 - k) : (S.tail_t0 + k);
            if (!row(i, 0, 1)) return;
        }
        return;
    }
    const i32 *rows = tail_on ? S.rows_nt : S.rows;
    // L with the tail on CTA 0: the tail rows' partial sums follow (tickets n_nt..)
    const unsigned total =
        (unsigned)(tail_on ? S.n_nt + (S.upper ? 0 : S.n_tail) : S.n) * (unsigned)S.nrhs;
    const int b0 = tail_on ? 1 : 0;  // CTA 0 is the tail's
    const unsigned nw = (gridDim.x - b0) * kWarps;
    const unsigned tb = S.tblock > 0 ? (unsigned)S.tblock : 1u;
    // tasks [t, t_end): a block of tb tickets (dynamic) or one task (static)
    unsigned t = 0, t_end = 0;
    if (S.tblock > 0) {
        if (lane == 0) t = atomicAdd(S.ticket, tb);
        t = __shfl_sync(0xffffffffu, t, 0);
    } else {
        t = (blockIdx.x - b0) * kWarps + w;
    }
    t_end = t + tb;
    while (t < total) {
        unsigned tn = 0;  // next block of tickets, in flight while this block runs
        if (S.tblock > 0 && t + 1 == t_end && lane == 0) tn = atomicAdd(S.ticket, tb);
        const int ri = (int)(t / (unsigned)S.nrhs), r = (int)(t % (unsigned)S.nrhs);
        const int i = (tail_on && ri >= S.n_nt) ? S.tail_t0 + (ri - S.n_nt) : __ldg(rows + ri);
        if (!row(i, r, (tail_on && ri >= S.n_nt) ? 2 : 0)) return;
        if (S.tblock == 0) {
            t += nw;
        } else if (++t == t_end) {
            t = __shfl_sync(0xffffffffu, tn, 0);
            t_end = t + tb;
        }
    }
}

// Several right-hand sides, on interleaved vectors (group g of 32
// right-hand sides, row c, lane l at ((g * n + c) * 32 + l)).  The host
// builds a level-ordered task list per k: a short row is ONE task per group
// of 32 right-hand sides -- lane l owns right-hand side 32g + l and runs its
// own chain, the row's indices and values are loaded once per chunk and
// shared through shared memory; a long row (more than kSolveLongRow entries,
// where that chain's per-chunk load latency would sit on the critical path)
// is one task PER right-hand side in the single-RHS form (lanes over
// entries, operands one chunk ahead).  Either way every column keeps the
// reference's per-element order: bitwise the single solve.
constexpr int kSolveLongRow = 96;

struct SolveTask {
    i32 row;
    i32 sub;  // >= 0: one right-hand side (long row); < 0: group -sub-1 (short row)
};

__global__ void __launch_bounds__(kThreads, 1) solve_dfm_kernel(SolveDfParams S, const SolveTask *tasks,
                                                                unsigned n_tasks) {
    __shared__ __align__(16) double vbuf[kWarps][32];
    __shared__ int icol[kWarps][kSolveRing][32], islot[kWarps][kSolveRing][32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const unsigned nw = gridDim.x * kWarps;
    unsigned t = 0;
    if (S.tblock > 0) {
        if (lane == 0) t = atomicAdd(S.ticket, 1u);
        t = __shfl_sync(0xffffffffu, t, 0);
    } else {
        t = blockIdx.x * kWarps + w;
    }
    while (t < n_tasks) {
        unsigned tn = 0;
        if (S.tblock > 0 && lane == 0) tn = atomicAdd(S.ticket, 1u);
        const SolveTask tk = tasks[t];
        const int i = tk.row;
        const bool per_rhs = tk.sub >= 0;
        const int grp = per_rhs ? (tk.sub >> 5) : (-tk.sub - 1);
        // this thread's right-hand side: the task's one (long row) or lane's (short row)
        const int r = per_rhs ? tk.sub : grp * 32 + lane;
        const int rl = r & 31;  // its lane within the interleaved group
        const bool active = r < S.nrhs;
        const double *Xg = S.out + (size_t)grp * S.n * 32 + rl;  // row c at Xg[c * 32]
        const int e0 = __ldg(S.ent_ptr + i), e1 = __ldg(S.ent_ptr + i + 1);
        const size_t own = ((size_t)grp * S.n + i) * 32 + rl;
        double acc = 0.0;
        if (active && (!per_rhs || lane == 0))
            acc = ldv(S.in_il ? S.in + own : S.in + (size_t)r * S.ld_in + i);
        const int ne = e1 - e0, ng = (ne + 31) >> 5;
        auto ent = [&](int k) { return S.upper ? (e1 - 1 - k) : (e0 + k); };
        auto issue_idx = [&](int g) {
            const int k = 32 * g + lane;
            const int e = ent(min(k, ne - 1));
            cp_async4(&icol[w][g % kSolveRing][lane], S.ent_col + e, k < ne);
            cp_async4(&islot[w][g % kSolveRing][lane], S.ent_slot + e, k < ne);
            cp_async_commit();
        };
        bool dead = false;
        if (ne > 0) {
#pragma unroll
            for (int g = 0; g < kSolveRing; ++g) issue_idx(g);
            if (per_rhs) {
                // lanes over entries, operands one chunk ahead, lane 0 chains
                unsigned long long xa = 0;
                double va = 0.0;
                cp_async_wait<kSolveRing - 1>();
                __syncwarp();
                if (lane < ne) {
                    xa = ld_relaxed_u64(Xg + (size_t)icol[w][0][lane] * 32);
                    va = ldv(S.v + islot[w][0][lane]);
                }
                for (int g = 0; g < ng && !dead; ++g) {
                    unsigned long long xb = 0;
                    double vb = 0.0;
                    cp_async_wait<kSolveRing - 2>();
                    __syncwarp();
                    const bool live = 32 * g + lane < ne;
                    if (__any_sync(0xffffffffu, live && xa == kSent)) {
                        const unsigned long long t0 = globaltimer();
                        const int c = icol[w][g % kSolveRing][lane];
                        while (true) {
                            const bool pend = live && xa == kSent;
                            if (!__any_sync(0xffffffffu, pend)) break;
                            if (pend) xa = ld_relaxed_u64(Xg + (size_t)c * 32);
                            if (__shfl_sync(0xffffffffu, globaltimer() - t0 > kWatchdogNs, 0)) {
                                dead = true;
                                break;
                            }
                        }
                    }
                    if (32 * (g + 1) + lane < ne) {
                        xb = ld_relaxed_u64(Xg + (size_t)icol[w][(g + 1) % kSolveRing][lane] * 32);
                        vb = ldv(S.v + islot[w][(g + 1) % kSolveRing][lane]);
                    }
                    __syncwarp();
                    issue_idx(g + kSolveRing);
                    const double x = __longlong_as_double((long long)xa);
                    const bool use = live && (S.upper ? true : (x != 0.0));
                    vbuf[w][lane] = use ? __dmul_rn(va, x) : 0.0;
                    __syncwarp();
                    if (lane == 0) {
                        const double2 *pb = reinterpret_cast<const double2 *>(vbuf[w]);
                        const int cnt = min(32, ne - 32 * g);
                        if (cnt == 32) {
#pragma unroll
                            for (int s2 = 0; s2 < 16; ++s2) {
                                const double2 p2 = pb[s2];
                                acc = __dsub_rn(acc, p2.x);
                                acc = __dsub_rn(acc, p2.y);
                            }
                        } else {
                            for (int s1 = 0; s1 < cnt; ++s1) acc = __dsub_rn(acc, vbuf[w][s1]);
                        }
                    }
                    __syncwarp();
                    xa = xb;
                    va = vb;
                }
            } else {
                // lanes over right-hand sides
                for (int g = 0; g < ng && !dead; ++g) {
                    cp_async_wait<kSolveRing - 1>();
                    __syncwarp();
                    const int sl = g % kSolveRing;
                    const int cnt = min(32, ne - 32 * g);
                    vbuf[w][lane] = lane < cnt ? ldv(S.v + islot[w][sl][lane]) : 0.0;
                    unsigned long long xs[32];
#pragma unroll
                    for (int e = 0; e < 32; ++e)
                        xs[e] = (active && e < cnt) ? ld_relaxed_u64(Xg + (size_t)icol[w][sl][e] * 32)
                                                    : 0ull;
                    __syncwarp();
                    bool pend = false;
#pragma unroll
                    for (int e = 0; e < 32; ++e) pend |= xs[e] == kSent;
                    if (__any_sync(0xffffffffu, pend)) {  // some inputs not done yet
                        const unsigned long long t0 = globaltimer();
                        while (true) {
                            pend = false;
#pragma unroll
                            for (int e = 0; e < 32; ++e)
                                if (xs[e] == kSent) {
                                    xs[e] = ld_relaxed_u64(Xg + (size_t)icol[w][sl][e] * 32);
                                    pend = true;
                                }
                            if (!__any_sync(0xffffffffu, pend)) break;
                            if (__shfl_sync(0xffffffffu, globaltimer() - t0 > kWatchdogNs, 0)) {
                                dead = true;
                                break;
                            }
                        }
                    }
                    // products first (independent), then the ordered chain
#pragma unroll
                    for (int e = 0; e < 32; ++e) {
                        const double x = __longlong_as_double((long long)xs[e]);
                        const bool use = e < cnt && (S.upper ? true : (x != 0.0));
                        xs[e] = (unsigned long long)__double_as_longlong(use ? __dmul_rn(vbuf[w][e], x) : 0.0);
                    }
#pragma unroll
                    for (int e = 0; e < 32; ++e) acc = __dsub_rn(acc, __longlong_as_double((long long)xs[e]));
                    __syncwarp();
                    issue_idx(g + kSolveRing);  // refill the slot of chunk g
                }
            }
            cp_async_wait<0>();
            __syncwarp();
        }
        if (dead) {  // warp-uniform
            if (lane == 0) atomicExch(S.err, 1u);
            return;
        }
        if (active && (!per_rhs || lane == 0)) {
            if (S.upper) acc = __ddiv_rn(acc, ldv(S.v + __ldg(S.diag_pos + i)));
            unsigned long long bits = (unsigned long long)__double_as_longlong(acc);
            if (bits == kSent) bits |= kQuietBit;
            st_relaxed_u64(S.out + own, bits);
            if (S.reset)
                st_relaxed_u64(S.reset_il ? S.reset + own : S.reset + (size_t)r * S.ld_reset + i, kSent);
        }
        if (S.tblock == 0) t += nw;
        else t = __shfl_sync(0xffffffffu, tn, 0);
    }
}

// dst[r][i] = src[r][i]; src[r][i] = sentinel (moves a vector into or out of
// the sentinel-managed buffers for the L-only / U-only entry points)
__global__ void solve_move_kernel(double *src, long long ld_src, double *dst, long long ld_dst,
                                  i32 n, i32 nrhs) {
    const long long total = (long long)n * nrhs;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < total;
         k += (long long)gridDim.x * blockDim.x) {
        const long long r = k / n, i = k % n;
        dst[r * ld_dst + i] = src[r * ld_src + i];
        src[r * ld_src + i] = __longlong_as_double((long long)kSent);
    }
}

// the same between the caller's layout (vector r at base + r * ld) and the
// interleaved one of the multi-RHS kernel
__device__ __forceinline__ double *vec_at(double *base, long long ld, int il, i32 n, long long r,
                                          long long i) {
    return il ? base + ((r >> 5) * n + i) * 32 + (r & 31) : base + r * ld + i;
}

__global__ void solve_xmove_kernel(double *src, long long ld_src, int il_src, double *dst,
                                   long long ld_dst, int il_dst, i32 n, i32 nrhs) {
    const long long total = (long long)n * nrhs;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < total;
         k += (long long)gridDim.x * blockDim.x) {
        const long long i = k / nrhs, r = k % nrhs;
        double *ps = vec_at(src, ld_src, il_src, n, r, i);
        *vec_at(dst, ld_dst, il_dst, n, r, i) = *ps;
        *ps = __longlong_as_double((long long)kSent);
    }
}

// batched launches: OR each launch's watchdog word into a sticky one (the
// next launch's memset clears the per-launch word)
__global__ void err_or_kernel(int *acc, const int *err) { *acc |= *err; }

__global__ void fill_sentinel_kernel(double *p, long long m) {
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < m;
         k += (long long)gridDim.x * blockDim.x)
        p[k] = __longlong_as_double((long long)kSent);
}

// per set: the largest column with an exactly zero diagonal (the column the
// reference's reverse sweep stops at, _kernels.py:186-197), or -1
__global__ void zero_pivot_batch_kernel(const double *v, long long stride, const i32 *diag_pos, i32 n,
                                        int nb, int *fail) {
    const long long total = (long long)n * nb;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < total;
         k += (long long)gridDim.x * blockDim.x) {
        const int b = (int)(k / n), j = (int)(k % n);
        if (v[(size_t)b * stride + diag_pos[j]] == 0.0) atomicMax(fail + b, j);
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
    i32 *level_need = nullptr;  // per phase: item count
    i32 *col_total = nullptr;   // per column: items into it
    glu::ColDep *cdeps = nullptr;
    i64 tail_t0 = 0;            // dense cluster tail: columns [tail_t0, n)
    i64 max_push_macs = 0;  // largest push item of the plan (kernel variant)
    TailShape tail;
    double *tail_g = nullptr;
    unsigned long long *tail_mk = nullptr;  // structure bitmasks of the tail columns
    i32 *tail_blk = nullptr;                // per tail column: first slot inside the block
    double *tail_umax = nullptr;            // per tail column: max |U| above the block (scratch)
    unsigned long long *fail_batch = nullptr;
    i64 fail_batch_cap = 0;
    // optional per-launch kernel timing: a ring of event triples
    std::vector<cudaEvent_t> kev;
    i64 kev_slots = 0, kev_next = 0;
    unsigned *sync = nullptr;   // done[n_levels*8] | err (+pad) | col_done[n]
    size_t sync_words = 0;
    Item *items = nullptr;
    Chunk *chunks = nullptr;
    uint8_t *map8 = nullptr;
    uint16_t *tgt16 = nullptr;
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
    int *ifail = nullptr;
    int *err_acc = nullptr;  // sticky watchdog word across the launches of one batched call
    // dataflow solves: sentinel-managed y buffer, [ticket, err] words
    double *solve_y = nullptr;
    i64 solve_y_cap = 0;
    unsigned *sctl = nullptr;
    int solve_tblock = 1;  // dataflow solve: tickets per grab (0 = static round-robin)
    bool solve_multi = true;  // k > 1: lanes over right-hand sides (solve_dfm_kernel)
    double *solve_yi = nullptr, *solve_zi = nullptr;  // interleaved y / x, sentinel between calls
    i64 solve_il_cap = 0;
    // multi-RHS task lists (level order; built per k)
    std::vector<i32> l_rows_h, u_rows_h, l_ptr_h, u_ptr_h;
    i32 *l_rows_nt = nullptr, *u_rows_nt = nullptr;  // level order without the dense-tail rows
    i32 *l_split = nullptr;        // L tail row: first entry in a tail column
    double *solve_part = nullptr;  // L tail rows' partial sums (sentinel between calls)
    i64 n_rows_nt = 0;
    bool solve_tail = true;  // option 14
    SolveTask *tasks_l = nullptr, *tasks_u = nullptr;
    unsigned n_tasks_l = 0, n_tasks_u = 0;
    int tasks_k = 0;
    int solve_long_row = kSolveLongRow;
    unsigned long long *tail_trace = nullptr;  // option 13
    unsigned long long *level_ns = nullptr;
    std::vector<i64> level_item_ptr_h;
    unsigned long long *trace = nullptr;
    i64 trace_l0 = 0, trace_nl = 0, trace_cap = 0;
    bool time_levels = false;
    bool fail_by_column = false;
    int poll_ns = 32;
    std::vector<double> last_level_ms;
    // host-API staging
    double *d_a = nullptr, *d_v = nullptr, *d_x = nullptr;
    double *d_ab = nullptr, *d_vb = nullptr;  // batched host-API staging
    cudaEvent_t ev_main = nullptr, ev_copy = nullptr;  // host API: overlap the D2H copy with the tail
    cudaStream_t stream2 = nullptr;
    i64 col_ptr_h_t0 = 0;  // first slot of the dense tail
    cudaStream_t stream = nullptr;
    glu::SnDev *sn = nullptr;  // supernodal engine (plans from glu_plan_build_sn)
};

namespace {

template <class T>
i64 track_upload(glu_handle *h, T **dst, const std::vector<T> &src) {
    GLU_CUDA(upload(dst, src));
    h->bytes += (i64)(src.size() * sizeof(T));
    return GLU_OK;
}

template <class T>
i64 upload_raw(glu_handle *h, T **dst, const T *src, i64 count) {
    *dst = nullptr;
    if (count <= 0) return GLU_OK;
    const size_t bytes = (size_t)count * sizeof(T);
    if (cudaMalloc((void **)dst, bytes) != cudaSuccess) {
        glu::set_error("cudaMalloc(" + std::to_string(bytes) + " B) for the update plan");
        return GLU_ECUDA;
    }
    GLU_CUDA(cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice));
    h->bytes += (i64)bytes;
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

constexpr size_t kFactorDynSmem = sizeof(int4) * kWarps * kDeepRing * 32;

int coop_grid(const void *kernel, int sm_count, size_t dyn_smem = 0) {
    int per_sm = 0;
    if (dyn_smem > 0 &&
        cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn_smem) != cudaSuccess)
        return 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThreads, dyn_smem) != cudaSuccess)
        return 0;
    per_sm = std::min(per_sm, 1);
    return per_sm * sm_count;
}

}  // namespace

// Every entry point runs on the handle's device, whatever the caller's
// current device is (restored on return).
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(const glu_handle *h) {
        if (cudaGetDevice(&prev) == cudaSuccess && prev != h->device) cudaSetDevice(h->device);
        else prev = -1;
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

extern "C" const char *glu_version(void) { return "glu_b200 0.1 sm_100a"; }

extern "C" int64_t glu_tail_capacity(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        return 0;
    }
    int cap = 0;
    pick_tail(0, &cap);
    return cap;
}

extern "C" void *glu_host_alloc(int64_t nbytes) {
    void *p = nullptr;
    const cudaError_t e = cudaHostAlloc(&p, (size_t)std::max<int64_t>(nbytes, 8), cudaHostAllocPortable);
    if (e != cudaSuccess) {
        cudaGetLastError();
        glu::set_error(std::string("glu_host_alloc: ") + cudaGetErrorString(e));
        return nullptr;
    }
    return p;
}

extern "C" void glu_host_free(void *p) {
    if (p) cudaFreeHost(p);
}

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
    {
        std::vector<i32> need(std::max<i64>(pv.n_levels, 1), 0);
        for (i64 l = 0; l < pv.n_levels; l++)
            need[l] = (i32)(pv.level_item_ptr[l + 1] - pv.level_item_ptr[l]);
        h->level_item_ptr_h.assign(pv.level_item_ptr, pv.level_item_ptr + pv.n_levels + 1);
        UP(h->level_need, need);
        h->sync_words = (size_t)std::max<i64>(pv.n_levels, 1) * 8 + kLineWords + (size_t)std::max<i64>(n, 1) * kColRep;
        UP(h->col_total, std::vector<i32>(pv.col_total, pv.col_total + n));
        if ((rc = upload_raw(h, &h->cdeps, pv.cdeps, pv.n_cdeps)) != GLU_OK) return fail(rc);
        h->tail_t0 = pv.tail_t0;
        h->col_ptr_h_t0 = col_ptr[pv.tail_t0];
        h->max_push_macs = pv.max_push_macs;
        const i64 m = n - pv.tail_t0;
        if (m > 0) {
            h->tail = pick_tail((int)m, nullptr);
            if (h->tail.C == 0) {
                glu::set_error("dense tail of " + std::to_string(m) +
                               " columns exceeds this device's cluster capacity (glu_tail_capacity)");
                return fail(GLU_EINVAL);
            }
            {  // per tail column: rows of the block present in the pattern
                const int mw = h->tail.mw;
                std::vector<unsigned long long> mk((size_t)m * mw, 0ull);
                for (i64 q = 0; q < m; q++)
                    for (i64 p = col_ptr[pv.tail_t0 + q]; p < col_ptr[pv.tail_t0 + q + 1]; p++) {
                        const i64 r = row_idx[p] - pv.tail_t0;
                        if (r >= 0) mk[(size_t)q * mw + (r >> 6)] |= 1ull << (r & 63);
                    }
                UP(h->tail_mk, mk);
                std::vector<i32> blk((size_t)m);
                for (i64 q = 0; q < m; q++) {
                    i64 p = col_ptr[pv.tail_t0 + q];
                    while (p < col_ptr[pv.tail_t0 + q + 1] && row_idx[p] < pv.tail_t0) p++;
                    blk[q] = (i32)p;
                }
                UP(h->tail_blk, blk);
                if (cudaMalloc((void **)&h->tail_umax, sizeof(double) * m * kMaxTailSets) != cudaSuccess) {
                    glu::set_error("cudaMalloc(tail maxima)");
                    return fail(GLU_ECUDA);
                }
            }
            if (cudaMalloc((void **)&h->tail_g, sizeof(double) * tail_set_doubles(h->tail) * kMaxTailSets) !=
                cudaSuccess) {
                glu::set_error("cudaMalloc(tail buffer)");
                return fail(GLU_ECUDA);
            }
        }
        if (cudaMalloc((void **)&h->sync, h->sync_words * sizeof(unsigned)) != cudaSuccess) {
            glu::set_error("cudaMalloc(sync)");
            return fail(GLU_ECUDA);
        }
    }
    UP(h->items, std::vector<Item>(pv.items, pv.items + pv.n_items));
    UP(h->chunks, std::vector<Chunk>(pv.chunks, pv.chunks + pv.n_chunks));
    UP(h->deep, std::vector<glu::DeepRef>(pv.deep, pv.deep + pv.n_deep));
    if ((rc = upload_raw(h, &h->map8, pv.map8, pv.n_map)) != GLU_OK) return fail(rc);
    if ((rc = upload_raw(h, &h->tgt16, pv.tgt16, pv.n_tgt)) != GLU_OK) return fail(rc);
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
    {
        std::vector<i32> lnt, unt;
        for (i32 i : lrows) if (i < h->tail_t0) lnt.push_back(i);
        for (i32 i : urows) if (i < h->tail_t0) unt.push_back(i);
        h->n_rows_nt = (i64)lnt.size();
        UP(h->l_rows_nt, lnt); UP(h->u_rows_nt, unt);
        const i64 mt = n - h->tail_t0;
        if (mt > 0) {
            std::vector<i32> split((size_t)mt);
            for (i64 k = 0; k < mt; k++) {
                const i64 i = h->tail_t0 + k;
                i32 e = lp[i];
                while (e < lp[i + 1] && lc[e] < h->tail_t0) e++;
                split[k] = e;
            }
            UP(h->l_split, split);
            if (cudaMalloc((void **)&h->solve_part, sizeof(double) * mt) != cudaSuccess) {
                glu::set_error("cudaMalloc(solve partials)");
                return fail(GLU_ECUDA);
            }
            fill_sentinel_kernel<<<4, 256>>>(h->solve_part, mt);
            if (cudaDeviceSynchronize() != cudaSuccess) { glu::set_error("fill"); return fail(GLU_ECUDA); }
        }
    }
    h->l_rows_h = std::move(lrows); h->u_rows_h = std::move(urows);
    h->l_ptr_h = std::move(lp); h->u_ptr_h = std::move(up_);
#undef UP
    if (cudaMalloc((void **)&h->fail, sizeof(unsigned long long)) != cudaSuccess ||
        cudaMalloc((void **)&h->ifail, sizeof(int)) != cudaSuccess ||
        cudaMalloc((void **)&h->err_acc, sizeof(int)) != cudaSuccess ||
        cudaMalloc((void **)&h->sctl, 2 * sizeof(unsigned)) != cudaSuccess) {
        glu::set_error("cudaMalloc(scratch)"); return fail(GLU_ECUDA);
    }
    if (pv.sn) {
        if ((rc = glu::sn_upload(pv.sn, &h->sn, &h->bytes)) != GLU_OK) return fail(rc);
    }
    h->grid = std::min({coop_grid((const void *)factor_kernel<4, 1>, h->sm_count, kFactorDynSmem),
                        coop_grid((const void *)factor_kernel<2, 2>, h->sm_count, kFactorDynSmem),
                        coop_grid((const void *)factor_kernel<2, 1>, h->sm_count, kFactorDynSmem),
                        coop_grid((const void *)solve_df_kernel, h->sm_count),
                        coop_grid((const void *)solve_dfm_kernel, h->sm_count)});
    if (h->grid <= 0) { glu::set_error("persistent kernel cannot be co-resident"); return fail(GLU_ECUDA); }
    *out = h;
    return GLU_OK;
}

extern "C" void glu_destroy(glu_handle *h) {
    if (!h) return;
    void *ptrs[] = {h->col_ptr, h->row_idx, h->diag_pos, h->level_of, h->level_need, h->col_total, h->cdeps, h->sync, h->tail_g, h->fail_batch, h->items,
                    h->chunks, h->map8, h->tgt16, h->deep, h->l_lvl_ptr, h->l_rows, h->l_ptr, h->l_col, h->l_slot,
                    h->u_lvl_ptr, h->u_rows, h->u_ptr, h->u_col, h->u_slot, h->a_slot, h->fail,
                    h->ifail, h->err_acc, h->tail_trace, h->tail_mk, h->tail_blk, h->tail_umax, h->solve_y, h->solve_yi, h->solve_zi, h->tasks_l, h->tasks_u, h->l_rows_nt, h->u_rows_nt, h->l_split, h->solve_part, h->sctl, h->level_ns, h->trace, h->d_a, h->d_v, h->d_x, h->d_ab, h->d_vb};
    for (void *p : ptrs)
        if (p) cudaFree(p);
    glu::sn_free(h->sn);
    if (h->stream) cudaStreamDestroy(h->stream);
    if (h->stream2) cudaStreamDestroy(h->stream2);
    if (h->ev_main) cudaEventDestroy(h->ev_main);
    if (h->ev_copy) cudaEventDestroy(h->ev_copy);
    for (cudaEvent_t e : h->kev) cudaEventDestroy(e);
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
        case 3:  // diagnostics: first traced phase
            h->trace_l0 = std::max<i64>(0, std::min<i64>(value, h->n_levels));
            return GLU_OK;
        case 4: {  // diagnostics: number of traced phases (0 = off)
            h->trace_nl = std::max<i64>(0, std::min<i64>(value, h->n_levels - h->trace_l0));
            const i64 cnt = h->level_item_ptr_h[h->trace_l0 + h->trace_nl] - h->level_item_ptr_h[h->trace_l0];
            if (cnt > h->trace_cap) {
                if (h->trace) cudaFree(h->trace);
                h->trace = nullptr;
                GLU_CUDA(cudaMalloc((void **)&h->trace, sizeof(unsigned long long) * 8 * cnt));
                h->trace_cap = cnt;
            }
            return GLU_OK;
        }
        case 6:  // tuning: nanoseconds between dependency polls
            h->poll_ns = (int)std::max<int64_t>(0, std::min<int64_t>(value, 100000));
            return GLU_OK;
        case 8: {  // diagnostics: record kernel times of the next `value` launches (ring)
            for (cudaEvent_t e : h->kev) cudaEventDestroy(e);
            h->kev.clear();
            h->kev_slots = std::max<int64_t>(0, value);
            h->kev_next = 0;
            h->kev.resize(3 * h->kev_slots);
            for (auto &e : h->kev) GLU_CUDA(cudaEventCreate(&e));
            return GLU_OK;
        }
        case 9:  // solves: 0 dataflow (the only solve kernel; the level-synchronous one was removed)
            if (value != 0) {
                glu::set_error("option 9: the level-synchronous solve kernel was removed (dataflow only)");
                return GLU_EINVAL;
            }
            return GLU_OK;
        case 11:  // tuning: k > 1 right-hand sides, 1 lanes over right-hand sides, 0 one warp each
            h->solve_multi = value != 0;
            return GLU_OK;
        case 13: {  // diagnostics: tail-kernel timestamps (glu_tail_trace_read)
            if (h->tail_trace) cudaFree(h->tail_trace);
            h->tail_trace = nullptr;
            if (value != 0 && h->tail.np > 0) {
                const size_t words = 8 + 6 * (size_t)h->tail.np;
                GLU_CUDA(cudaMalloc((void **)&h->tail_trace, sizeof(unsigned long long) * words));
                GLU_CUDA(cudaMemset(h->tail_trace, 0, sizeof(unsigned long long) * words));
            }
            return GLU_OK;
        }
        case 14:  // tuning: single-RHS solves keep the dense-tail rows on CTA 0 (default 1)
            h->solve_tail = value != 0;
            return GLU_OK;
        case 12:  // tuning: k > 1 solves, rows longer than this run one task per right-hand side
            h->solve_long_row = (int)std::max<int64_t>(0, std::min<int64_t>(value, 1 << 30));
            h->tasks_k = 0;  // rebuild the task lists
            return GLU_OK;
        case 10:  // tuning: dataflow-solve tasks per ticket grab (0 = static round-robin)
            h->solve_tblock = (int)std::max<int64_t>(0, std::min<int64_t>(value, 64));
            return GLU_OK;
        case 15:  // diagnostics: supernodal engine per-task timestamps (glu_sn_trace)
            if (!h->sn) { glu::set_error("option 15 needs a supernodal handle"); return GLU_EINVAL; }
            return glu::sn_set_trace(h->sn, (int)value);
        case 2:  // failing-pivot order: 0 level-major (factor_parallel), 1 column (sequential paths)
            h->fail_by_column = value != 0;
            return GLU_OK;
        default:
            glu::set_error("unknown option");
            return GLU_EINVAL;
    }
}

extern "C" int64_t glu_sn_trace(glu_handle *h, int64_t *out, int64_t max_tasks) {
    if (!h->sn) return 0;
    return glu::sn_read_trace(h->sn, out, max_tasks);
}

extern "C" int64_t glu_set_fail_levels(glu_handle *h, const int64_t *level_of) {
    std::vector<i32> lv = to_i32(level_of, h->n);
    if (!lv.empty())
        GLU_CUDA(cudaMemcpy(h->level_of, lv.data(), sizeof(i32) * lv.size(), cudaMemcpyHostToDevice));
    return GLU_OK;
}

extern "C" int64_t glu_kernel_times(glu_handle *h, double *ms, int64_t max_launches) {
    const i64 m = std::min<i64>({max_launches, h->kev_slots, h->kev_next});
    for (i64 k = 0; k < m; k++) {
        float a = 0.f, b = 0.f;
        GLU_CUDA(cudaEventElapsedTime(&a, h->kev[3 * k], h->kev[3 * k + 1]));
        GLU_CUDA(cudaEventElapsedTime(&b, h->kev[3 * k + 1], h->kev[3 * k + 2]));
        ms[2 * k] = a;
        ms[2 * k + 1] = b;
    }
    return m;
}

extern "C" int64_t glu_tail_trace_read(glu_handle *h, int64_t *out, int64_t max_words) {
    if (!h->tail_trace) return 0;
    const i64 words = std::min<i64>(max_words, 8 + 6 * (i64)h->tail.np);
    GLU_CUDA(cudaDeviceSynchronize());
    GLU_CUDA(cudaMemcpy(out, h->tail_trace, sizeof(int64_t) * words, cudaMemcpyDeviceToHost));
    return words;
}

extern "C" int64_t glu_trace_read(glu_handle *h, int64_t *out, int64_t max_records) {
    if (h->trace_nl <= 0 || !h->trace) return 0;
    const i64 cnt = h->level_item_ptr_h[h->trace_l0 + h->trace_nl] - h->level_item_ptr_h[h->trace_l0];
    const i64 m = std::min<i64>(cnt, max_records);
    if (m > 0) GLU_CUDA(cudaMemcpy(out, h->trace, sizeof(unsigned long long) * 8 * m, cudaMemcpyDeviceToHost));
    return m;
}

extern "C" int64_t glu_level_times(const glu_handle *h, double *ms, int64_t len) {
    const i64 m = std::min<i64>(len, (i64)h->last_level_ms.size());
    for (i64 i = 0; i < m; i++) ms[i] = h->last_level_ms[i];
    return m;
}

extern "C" int64_t glu_set_input_pattern(glu_handle *h, int64_t nz, const int64_t *a_col_ptr,
                                         const int64_t *a_row_idx) {
    DeviceGuard dg_(h);
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
    // batched staging is sized from nz: drop it with the old pattern
    if (h->d_ab) { cudaFree(h->d_ab); h->d_ab = nullptr; }
    if (h->d_vb) { cudaFree(h->d_vb); h->d_vb = nullptr; }
    i64 rc = track_upload(h, &h->a_slot, slot);
    if (rc != GLU_OK) return rc;
    h->nz = nz;
    return GLU_OK;
}

extern "C" int64_t glu_scatter_device(glu_handle *h, const double *a_vals, double *v, void *stream) {
    DeviceGuard dg_(h);
    if (h->nz < 0) { glu::set_error("glu_set_input_pattern not called"); return GLU_EINVAL; }
    cudaStream_t s = (cudaStream_t)stream;
    const int blocks = h->sm_count * 4;
    zero_kernel<<<blocks, 256, 0, s>>>(v, h->nnz);
    if (h->nz > 0) scatter_kernel<<<blocks, 256, 0, s>>>(a_vals, h->a_slot, h->nz, v);
    GLU_CUDA(cudaGetLastError());
    return GLU_OK;
}

static int64_t launch_factor(glu_handle *h, double *v, double thresh, cudaStream_t s,
                             unsigned long long *fail = nullptr, int nb = 1) {
    if (!fail) fail = h->fail;
    if (nb > kMaxTailSets && h->tail_t0 < h->n) {
        glu::set_error("batched launch: at most 16 value sets per launch with a dense tail");
        return GLU_EINVAL;
    }
    GLU_CUDA(cudaMemsetAsync(fail, 0xff, sizeof(unsigned long long) * nb, s));
    if (h->sn) {  // supernodal engine: one launch (+ pivot-check pass) per value set
        const size_t nl8s = (size_t)std::max<i64>(h->n_levels, 1) * 8;
        cudaEvent_t *ke = nullptr;
        if (h->kev_slots > 0) {
            ke = &h->kev[3 * (h->kev_next % h->kev_slots)];
            h->kev_next++;
            GLU_CUDA(cudaEventRecord(ke[0], s));
        }
        GLU_CUDA(cudaMemsetAsync(h->sync + nl8s, 0, sizeof(int), s));  // watchdog word
        for (int b = 0; b < nb; b++) {
            const i64 rc = glu::sn_launch(h->sn, v + (size_t)b * h->nnz, h->col_ptr, h->diag_pos, h->level_of,
                                          (i32)h->n, thresh, h->fail_by_column, fail + b,
                                          (int *)(h->sync + nl8s), s);
            if (rc != GLU_OK) return rc;
        }
        if (ke) {
            GLU_CUDA(cudaEventRecord(ke[1], s));
            GLU_CUDA(cudaEventRecord(ke[2], s));
        }
        return GLU_OK;
    }
    GLU_CUDA(cudaMemsetAsync(h->sync, 0, h->sync_words * sizeof(unsigned), s));
    FactorParams P;
    P.v = v;
    P.items = h->items;
    P.chunks = h->chunks;
    P.map8 = h->map8;
    P.tgt16 = h->tgt16;
    P.deep = h->deep;
    P.col_ptr = h->col_ptr;
    P.diag_pos = h->diag_pos;
    P.level_of = h->level_of;
    P.level_need = h->level_need;
    P.n = (i32)h->n;
    P.n_items = (i32)h->n_items;
    P.n_levels = (i32)h->n_levels;
    P.n_div = (i32)h->tail_t0;
    P.nb = nb;
    P.set_stride = h->nnz;
    P.thresh = thresh;
    P.fail = fail;
    const size_t nl8 = (size_t)std::max<i64>(h->n_levels, 1) * 8;
    P.done = h->sync;
    P.col_done = h->sync + nl8 + kLineWords;
    P.col_total = h->col_total;
    P.cdeps = h->cdeps;
    P.err = (int *)(h->sync + nl8);
    P.level_ns = h->time_levels ? h->level_ns : nullptr;
    P.fail_by_column = h->fail_by_column ? 1 : 0;
    P.trace = nullptr;
    P.trace_i0 = P.trace_i1 = 0;
    P.poll_ns = h->poll_ns;
    if (h->trace_nl > 0 && h->trace) {
        P.trace = h->trace;
        P.trace_i0 = (i32)h->level_item_ptr_h[h->trace_l0];
        P.trace_i1 = (i32)h->level_item_ptr_h[h->trace_l0 + h->trace_nl];
        GLU_CUDA(cudaMemsetAsync(h->trace, 0, sizeof(unsigned long long) * 8 * (P.trace_i1 - P.trace_i0), s));
    }
    void *args[] = {&P};
    if (h->time_levels) {
        GLU_CUDA(cudaMemsetAsync(h->level_ns, 0, sizeof(unsigned long long) * (h->n_levels + 1), s));
    }
    cudaEvent_t *ke = nullptr;
    if (h->kev_slots > 0) {
        ke = &h->kev[3 * (h->kev_next % h->kev_slots)];
        h->kev_next++;
        GLU_CUDA(cudaEventRecord(ke[0], s));
    }
    // plans with <= 64-MAC items (batch plans) run the 2-entries-per-lane
    // variant, which loads two value sets per round in batched launches
    const void *kfn = h->max_push_macs <= 64 ? (nb > 1 ? (const void *)factor_kernel<2, 2>
                                                        : (const void *)factor_kernel<2, 1>)
                                             : (const void *)factor_kernel<4, 1>;
    GLU_CUDA(cudaLaunchCooperativeKernel(kfn, dim3(h->grid), dim3(kThreads), args, kFactorDynSmem, s));
    if (ke) GLU_CUDA(cudaEventRecord(ke[1], s));
    if (h->ev_main) GLU_CUDA(cudaEventRecord(h->ev_main, s));  // columns < tail_t0 final
    if (h->tail_t0 < h->n) {
        TailParams T;
        T.v = v;
        T.col_ptr = h->col_ptr;
        T.row_idx = h->row_idx;
        T.diag_pos = h->diag_pos;
        T.level_of = h->level_of;
        T.t0 = (i32)h->tail_t0;
        T.m = (i32)(h->n - h->tail_t0);
        T.mpad = h->tail.mpad;
        T.mw = h->tail.mw;
        T.b = h->tail.b;
        T.np = h->tail.np;
        T.ncl = h->tail.ncl;
        T.gstride = tail_gstride(h->tail);
        T.G = h->tail_g;
        T.g_set = tail_set_doubles(h->tail);
        T.set_stride = h->nnz;
        T.ready = reinterpret_cast<unsigned *>(h->tail_g + (size_t)h->tail.np * T.gstride);
        for (int b = 0; b < nb; ++b)  // every set's panel flags
            GLU_CUDA(cudaMemsetAsync(reinterpret_cast<unsigned *>(h->tail_g + (size_t)b * T.g_set +
                                                                  (size_t)h->tail.np * T.gstride),
                                     0, sizeof(unsigned) * h->tail.np, s));
        T.thresh = thresh;
        T.fail = fail;
        T.fail_by_column = h->fail_by_column ? 1 : 0;
        T.trace = h->tail_trace;
        T.mk0 = h->tail_mk;
        T.blk = h->tail_blk;
        T.umax = h->tail_umax;
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = h->tail.C;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(h->tail.C * nb);  // one cluster per value set
        cfg.blockDim = dim3(kTailThreads);
        cfg.dynamicSmemBytes = h->tail.smem;
        cfg.stream = s;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        GLU_CUDA(cudaLaunchKernelEx(&cfg, tail_kernel, T));
    }
    if (ke) GLU_CUDA(cudaEventRecord(ke[2], s));
    return GLU_OK;
}

static int64_t read_fail(glu_handle *h, cudaStream_t s) {
    unsigned long long key = 0;
    int err = 0;
    const size_t nl8 = (size_t)std::max<i64>(h->n_levels, 1) * 8;
    GLU_CUDA(cudaMemcpyAsync(&key, h->fail, sizeof(key), cudaMemcpyDeviceToHost, s));
    GLU_CUDA(cudaMemcpyAsync(&err, h->sync + nl8, sizeof(int),
                             cudaMemcpyDeviceToHost, s));
    GLU_CUDA(cudaStreamSynchronize(s));
    if (err) {
        glu::set_error("factor kernel watchdog: a phase dependency wait exceeded 4 s");
        return GLU_ECUDA;
    }
    if (h->time_levels && h->n_levels > 0) {
        std::vector<unsigned long long> ns(h->n_levels + 1);
        GLU_CUDA(cudaMemcpy(ns.data(), h->level_ns, sizeof(unsigned long long) * (h->n_levels + 1),
                            cudaMemcpyDeviceToHost));
        // phases without items never complete on their own: carry the time forward
        for (i64 l = 1; l <= h->n_levels; l++)
            if (ns[l] == 0) ns[l] = ns[l - 1];
        h->last_level_ms.assign(h->n_levels, 0.0);
        for (i64 l = 0; l < h->n_levels; l++) h->last_level_ms[l] = (double)(ns[l + 1] - ns[l]) * 1e-6;
    }
    if (key == ~0ull) return GLU_OK;
    return (int64_t)(key & 0xffffffffull);
}

extern "C" int64_t glu_factor_device(glu_handle *h, double *v, double thresh, void *stream) {
    DeviceGuard dg_(h);
    cudaStream_t s = (cudaStream_t)stream;
    i64 rc = launch_factor(h, v, thresh, s);
    if (rc != GLU_OK) return rc;
    return read_fail(h, s);
}

// Asynchronous variant for timing loops: no host sync, no status read.
extern "C" int64_t glu_factor_device_async(glu_handle *h, double *v, double thresh, void *stream) {
    DeviceGuard dg_(h);
    return launch_factor(h, v, thresh, (cudaStream_t)stream);
}

extern "C" int64_t glu_factor_status(glu_handle *h, void *stream) {
    DeviceGuard dg_(h);
    return read_fail(h, (cudaStream_t)stream);
}

static int64_t ensure_staging(glu_handle *h);

// Batch refactorization (cfg5: many value sets on one pattern, e.g. the
// Newton / transient steps of a circuit simulation).  Value sets are
// batch-major (set b at v + b * nnz); every set is factored in stream order
// by the same resident plan, each with its own failure slot, and the
// statuses are read back once for the whole batch.
constexpr int kMaxBatchPerLaunch = 16;  // 8: 322 /s, 16: 343 /s, 32: 341 /s (cfg2)

static int64_t ensure_batch(glu_handle *h, int64_t batch) {
    if (batch <= h->fail_batch_cap) return GLU_OK;
    if (h->fail_batch) cudaFree(h->fail_batch);
    h->fail_batch = nullptr;
    GLU_CUDA(cudaMalloc((void **)&h->fail_batch, sizeof(unsigned long long) * batch));
    h->fail_batch_cap = batch;
    return GLU_OK;
}

static int64_t batch_status(glu_handle *h, int64_t batch, int64_t *fail_cols, cudaStream_t s) {
    std::vector<unsigned long long> keys((size_t)batch);
    int err = 0;
    const size_t nl8 = (size_t)std::max<i64>(h->n_levels, 1) * 8;
    GLU_CUDA(cudaMemcpyAsync(keys.data(), h->fail_batch, sizeof(unsigned long long) * batch,
                             cudaMemcpyDeviceToHost, s));
    (void)nl8;
    GLU_CUDA(cudaMemcpyAsync(&err, h->err_acc, sizeof(int), cudaMemcpyDeviceToHost, s));
    GLU_CUDA(cudaStreamSynchronize(s));
    if (err) {
        glu::set_error("factor kernel watchdog: a phase dependency wait exceeded 4 s");
        return GLU_ECUDA;
    }
    for (int64_t b = 0; b < batch; b++)
        fail_cols[b] = keys[b] == ~0ull ? GLU_OK : (int64_t)(keys[b] & 0xffffffffull);
    return GLU_OK;
}

extern "C" int64_t glu_factor_batch_device(glu_handle *h, int64_t batch, double *v, double thresh,
                                           int64_t *fail_cols, void *stream) {
    DeviceGuard dg_(h);
    if (batch < 0 || (batch > 0 && (!v || !fail_cols))) { glu::set_error("bad batch arguments"); return GLU_EINVAL; }
    cudaStream_t s = (cudaStream_t)stream;
    i64 rc = ensure_batch(h, std::max<int64_t>(batch, 1));
    if (rc != GLU_OK) return rc;
    // up to 16 sets per launch: they share each item's static loads,
    // dependency wait and release; a dense tail runs one cluster per set
    const size_t nl8 = (size_t)std::max<i64>(h->n_levels, 1) * 8;
    GLU_CUDA(cudaMemsetAsync(h->err_acc, 0, sizeof(int), s));
    for (int64_t b0 = 0; b0 < batch; b0 += kMaxBatchPerLaunch) {
        const int nb = (int)std::min<int64_t>(kMaxBatchPerLaunch, batch - b0);
        if ((rc = launch_factor(h, v + b0 * h->nnz, thresh, s, h->fail_batch + b0, nb)) != GLU_OK) return rc;
        err_or_kernel<<<1, 1, 0, s>>>(h->err_acc, (const int *)(h->sync + nl8));
    }
    return batch_status(h, batch, fail_cols, s);
}

extern "C" int64_t glu_factor_batch_host(glu_handle *h, int64_t batch, const double *a_vals,
                                         double *lu_out, double thresh, int64_t *fail_cols) {
    DeviceGuard dg_(h);
    if (h->nz < 0) { glu::set_error("glu_set_input_pattern not called"); return GLU_EINVAL; }
    if (batch < 0 || (batch > 0 && (!a_vals || !lu_out || !fail_cols))) {
        glu::set_error("bad batch arguments");
        return GLU_EINVAL;
    }
    i64 rc = ensure_staging(h);
    if (rc != GLU_OK) return rc;
    if ((rc = ensure_batch(h, std::max<int64_t>(batch, 1))) != GLU_OK) return rc;
    cudaStream_t s = h->stream;
    const bool batched = true;  // sets share a launch (a dense tail: one cluster per set)
    const int chunk = batched ? kMaxBatchPerLaunch : 1;
    if (batched && !h->d_vb) {
        GLU_CUDA(cudaMalloc((void **)&h->d_vb, sizeof(double) * h->nnz * chunk));
        GLU_CUDA(cudaMalloc((void **)&h->d_ab, sizeof(double) * std::max<i64>(h->nz, 1) * chunk));
    }
    double *dv = batched ? h->d_vb : h->d_v, *da = batched ? h->d_ab : h->d_a;
    const size_t nl8 = (size_t)std::max<i64>(h->n_levels, 1) * 8;
    GLU_CUDA(cudaMemsetAsync(h->err_acc, 0, sizeof(int), s));
    for (int64_t b0 = 0; b0 < batch; b0 += chunk) {
        const int nb = (int)std::min<int64_t>(chunk, batch - b0);
        GLU_CUDA(cudaMemcpyAsync(da, a_vals + b0 * h->nz, sizeof(double) * h->nz * nb,
                                 cudaMemcpyHostToDevice, s));
        for (int k = 0; k < nb; k++)
            if ((rc = glu_scatter_device(h, da + (size_t)k * h->nz, dv + (size_t)k * h->nnz, s)) != GLU_OK)
                return rc;
        if ((rc = launch_factor(h, dv, thresh, s, h->fail_batch + b0, nb)) != GLU_OK) return rc;
        err_or_kernel<<<1, 1, 0, s>>>(h->err_acc, (const int *)(h->sync + nl8));
        GLU_CUDA(cudaMemcpyAsync(lu_out + b0 * h->nnz, dv, sizeof(double) * h->nnz * nb,
                                 cudaMemcpyDeviceToHost, s));
    }
    return batch_status(h, batch, fail_cols, s);
}

// y scratch of the dataflow solves, all-sentinel between calls
static int64_t ensure_solve_y(glu_handle *h, int nrhs, cudaStream_t s) {
    const i64 need = std::max<i64>(h->n, 1) * nrhs;
    if (need <= h->solve_y_cap) return GLU_OK;
    GLU_CUDA(cudaStreamSynchronize(s));
    if (h->solve_y) cudaFree(h->solve_y);
    h->solve_y = nullptr;
    h->solve_y_cap = 0;
    GLU_CUDA(cudaMalloc((void **)&h->solve_y, sizeof(double) * need));
    fill_sentinel_kernel<<<h->sm_count * 4, 256, 0, s>>>(h->solve_y, need);
    GLU_CUDA(cudaGetLastError());
    h->solve_y_cap = need;
    return GLU_OK;
}

static int64_t ensure_solve_il(glu_handle *h, int nrhs, cudaStream_t s) {
    const i64 need = std::max<i64>(h->n, 1) * (i64)((nrhs + 31) / 32) * 32;
    if (need <= h->solve_il_cap) return GLU_OK;
    GLU_CUDA(cudaStreamSynchronize(s));
    for (double **p : {&h->solve_yi, &h->solve_zi}) {
        if (*p) cudaFree(*p);
        *p = nullptr;
    }
    h->solve_il_cap = 0;
    GLU_CUDA(cudaMalloc((void **)&h->solve_yi, sizeof(double) * need));
    GLU_CUDA(cudaMalloc((void **)&h->solve_zi, sizeof(double) * need));
    fill_sentinel_kernel<<<h->sm_count * 4, 256, 0, s>>>(h->solve_yi, need);
    fill_sentinel_kernel<<<h->sm_count * 4, 256, 0, s>>>(h->solve_zi, need);
    GLU_CUDA(cudaGetLastError());
    h->solve_il_cap = need;
    return GLU_OK;
}

static int64_t ensure_solve_tasks(glu_handle *h, int nrhs, cudaStream_t s) {
    if (h->tasks_k == nrhs) return GLU_OK;
    GLU_CUDA(cudaStreamSynchronize(s));
    for (SolveTask **p : {&h->tasks_l, &h->tasks_u}) {
        if (*p) cudaFree(*p);
        *p = nullptr;
    }
    h->tasks_k = 0;
    const int groups = (nrhs + 31) / 32;
    auto build = [&](const std::vector<i32> &rows, const std::vector<i32> &ptr, SolveTask **dst,
                     unsigned *cnt) -> int64_t {
        std::vector<SolveTask> t;
        t.reserve(rows.size() * groups);
        for (i32 i : rows) {
            if (ptr[i + 1] - ptr[i] > h->solve_long_row)
                for (int r = 0; r < nrhs; r++) t.push_back({i, r});
            else
                for (int g = 0; g < groups; g++) t.push_back({i, -(g + 1)});
        }
        if (t.size() >= (size_t)UINT32_MAX) {
            glu::set_error("too many solve tasks");
            return GLU_EINVAL;
        }
        *cnt = (unsigned)t.size();
        GLU_CUDA(upload(dst, t));
        return GLU_OK;
    };
    i64 rc;
    if ((rc = build(h->l_rows_h, h->l_ptr_h, &h->tasks_l, &h->n_tasks_l)) != GLU_OK) return rc;
    if ((rc = build(h->u_rows_h, h->u_ptr_h, &h->tasks_u, &h->n_tasks_u)) != GLU_OK) return rc;
    h->tasks_k = nrhs;
    return GLU_OK;
}

static void solve_params_common(glu_handle *h, SolveDfParams &S, const double *lu, bool upper, int nrhs) {
    S.v = lu;
    S.v_stride = 0;
    S.upper = upper ? 1 : 0;
    S.rows = upper ? h->u_rows : h->l_rows;
    S.ent_ptr = upper ? h->u_ptr : h->l_ptr;
    S.ent_col = upper ? h->u_col : h->l_col;
    S.ent_slot = upper ? h->u_slot : h->l_slot;
    S.diag_pos = h->diag_pos;
    S.n = (i32)h->n;
    S.nrhs = nrhs;
    S.tblock = h->solve_tblock;
    S.ticket = h->sctl;
    S.err = h->sctl + 1;
    S.in_il = S.reset_il = 0;
    const i64 m = h->n - h->tail_t0;
    // U pass only: its tail rows read only tail columns; an L tail row also
    // carries ~500 entries left of the block, and funnelling those through
    // one SM measured slower (cfg2 L 1.12 -> 1.66 ms, U 1.62 -> 1.47 ms)
    const bool tail = h->solve_tail && nrhs == 1 && m >= 128 && m <= kSolveTailMax && h->grid > 1;
    S.tail_t0 = (i32)h->tail_t0;
    S.n_tail = tail ? (i32)m : 0;
    S.n_nt = (i32)h->n_rows_nt;
    S.rows_nt = upper ? h->u_rows_nt : h->l_rows_nt;
    S.lsplit = h->l_split;
    S.part = h->solve_part;
}

// multi-RHS pass on the interleaved buffers: L reads x (caller layout) into
// yi; U reads yi (restoring it) into zi
static int64_t launch_solve_dfm(glu_handle *h, const double *lu, double *x, bool upper,
                                cudaStream_t s, int nrhs, i64 ldx) {
    SolveDfParams S;
    solve_params_common(h, S, lu, upper, nrhs);
    if (upper) {
        S.in = h->solve_yi; S.in_il = 1; S.ld_in = 0;
        S.out = h->solve_zi; S.ld_out = 0;
        S.reset = h->solve_yi; S.reset_il = 1; S.ld_reset = 0;
    } else {
        S.in = x; S.ld_in = ldx;
        S.out = h->solve_yi; S.ld_out = 0;
        S.reset = nullptr; S.ld_reset = 0;
    }
    const SolveTask *tasks = upper ? h->tasks_u : h->tasks_l;
    unsigned n_tasks = upper ? h->n_tasks_u : h->n_tasks_l;
    GLU_CUDA(cudaMemsetAsync(h->sctl, 0, sizeof(unsigned), s));
    void *args[] = {&S, &tasks, &n_tasks};
    GLU_CUDA(cudaLaunchCooperativeKernel((const void *)solve_dfm_kernel, dim3(h->grid), dim3(kThreads),
                                         args, 0, s));
    return GLU_OK;
}

static int64_t launch_solve_df(glu_handle *h, const double *lu, double *x, bool upper,
                               cudaStream_t s, int nrhs, i64 ldx, i64 v_stride = 0) {
    SolveDfParams S;
    solve_params_common(h, S, lu, upper, nrhs);
    S.v_stride = v_stride;
    if (v_stride != 0) S.n_tail = 0;  // batch solves: the per-set path
    if (upper) {
        S.in = h->solve_y; S.ld_in = h->n;
        S.out = x; S.ld_out = ldx;
        S.reset = h->solve_y; S.ld_reset = h->n;
    } else {
        S.in = x; S.ld_in = ldx;
        S.out = h->solve_y; S.ld_out = h->n;
        S.reset = x; S.ld_reset = ldx;
    }
    GLU_CUDA(cudaMemsetAsync(h->sctl, 0, sizeof(unsigned), s));
    void *args[] = {&S};
    GLU_CUDA(cudaLaunchCooperativeKernel((const void *)solve_df_kernel, dim3(h->grid), dim3(kThreads),
                                         args, 0, s));
    return GLU_OK;
}

// part 0 = L then U, 1 = L only, 2 = U only; x holds nrhs vectors at stride ldx.
static int64_t run_solves(glu_handle *h, const double *lu, double *x, int part, cudaStream_t s,
                          int nrhs = 1, i64 ldx = 0, i64 v_stride = 0) {
    if (ldx <= 0) ldx = h->n;
    i64 rc;
    if (h->n == 0) return GLU_OK;
    const int mg = h->sm_count * 4;
    GLU_CUDA(cudaMemsetAsync(h->sctl + 1, 0, sizeof(unsigned), s));
    if (nrhs > 1 && h->solve_multi && v_stride == 0) {
        if ((rc = ensure_solve_il(h, nrhs, s)) != GLU_OK) return rc;
        if ((rc = ensure_solve_tasks(h, nrhs, s)) != GLU_OK) return rc;
        const i32 n32 = (i32)h->n;
        if (part == 2) {  // y (caller layout) -> yi
            solve_xmove_kernel<<<mg, 256, 0, s>>>(x, ldx, 0, h->solve_yi, 0, 1, n32, nrhs);
            GLU_CUDA(cudaGetLastError());
        }
        if (part != 2 && (rc = launch_solve_dfm(h, lu, x, false, s, nrhs, ldx)) != GLU_OK) return rc;
        if (part != 1 && (rc = launch_solve_dfm(h, lu, x, true, s, nrhs, ldx)) != GLU_OK) return rc;
        double *res = part == 1 ? h->solve_yi : h->solve_zi;  // result -> x, buffer -> sentinel
        solve_xmove_kernel<<<mg, 256, 0, s>>>(res, 0, 1, x, ldx, 0, n32, nrhs);
        GLU_CUDA(cudaGetLastError());
    } else {
    if ((rc = ensure_solve_y(h, nrhs, s)) != GLU_OK) return rc;
    if (part == 2) {  // x (= y) into the y buffer, x to sentinel
        solve_move_kernel<<<mg, 256, 0, s>>>(x, ldx, h->solve_y, h->n, (i32)h->n, nrhs);
        GLU_CUDA(cudaGetLastError());
    }
    if (part != 2 && (rc = launch_solve_df(h, lu, x, false, s, nrhs, ldx, v_stride)) != GLU_OK) return rc;
    if (part != 1 && (rc = launch_solve_df(h, lu, x, true, s, nrhs, ldx, v_stride)) != GLU_OK) return rc;
    if (part == 1) {  // y back into x, the y buffer to sentinel
        solve_move_kernel<<<mg, 256, 0, s>>>(h->solve_y, h->n, x, ldx, (i32)h->n, nrhs);
        GLU_CUDA(cudaGetLastError());
    }
    }
    unsigned err = 0;
    GLU_CUDA(cudaMemcpyAsync(&err, h->sctl + 1, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
    GLU_CUDA(cudaStreamSynchronize(s));
    if (err) {
        if (h->solve_y) fill_sentinel_kernel<<<mg, 256, 0, s>>>(h->solve_y, h->solve_y_cap);
        if (h->solve_yi) fill_sentinel_kernel<<<mg, 256, 0, s>>>(h->solve_yi, h->solve_il_cap);
        if (h->solve_zi) fill_sentinel_kernel<<<mg, 256, 0, s>>>(h->solve_zi, h->solve_il_cap);
        if (h->solve_part) fill_sentinel_kernel<<<mg, 256, 0, s>>>(h->solve_part, h->n - h->tail_t0);
        cudaStreamSynchronize(s);
        glu::set_error("triangular solve: dependency wait exceeded the watchdog");
        return GLU_ECUDA;
    }
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
    DeviceGuard dg_(h);
    cudaStream_t s = (cudaStream_t)stream;
    i64 rc = run_solves(h, lu, x, 1, s);
    if (rc != GLU_OK) return rc;
    GLU_CUDA(cudaStreamSynchronize(s));
    return GLU_OK;
}

extern "C" int64_t glu_upper_solve_device(glu_handle *h, const double *lu, double *x, void *stream) {
    DeviceGuard dg_(h);
    cudaStream_t s = (cudaStream_t)stream;
    i64 rc = check_zero_pivot(h, lu, s);
    if (rc != GLU_OK) return rc;
    rc = run_solves(h, lu, x, 2, s);
    if (rc != GLU_OK) return rc;
    GLU_CUDA(cudaStreamSynchronize(s));
    return GLU_OK;
}

extern "C" int64_t glu_solve_device(glu_handle *h, const double *lu, double *x, void *stream) {
    DeviceGuard dg_(h);
    cudaStream_t s = (cudaStream_t)stream;
    i64 rc = check_zero_pivot(h, lu, s);
    if (rc != GLU_OK) return rc;
    if ((rc = run_solves(h, lu, x, 0, s)) != GLU_OK) return rc;
    GLU_CUDA(cudaStreamSynchronize(s));
    return GLU_OK;
}

static int64_t ensure_staging(glu_handle *h) {
    if (!h->d_v) GLU_CUDA(cudaMalloc((void **)&h->d_v, sizeof(double) * std::max<i64>(h->nnz, 1)));
    if (!h->d_a) GLU_CUDA(cudaMalloc((void **)&h->d_a, sizeof(double) * std::max<i64>(h->nz, 1)));
    if (!h->d_x) GLU_CUDA(cudaMalloc((void **)&h->d_x, sizeof(double) * std::max<i64>(h->n, 1)));
    return GLU_OK;
}

// Multi-RHS solves: x holds nrhs right-hand sides, column r at
// x + r * ldx; part 0 = L then U, 1 = L only, 2 = U only.  Every level
// spreads its (row, right-hand side) pairs over the warps; the per-element
// order is the reference's, so every column is bitwise the single solve.
extern "C" int64_t glu_solve_multi_device(glu_handle *h, const double *lu, double *x, int64_t nrhs,
                                          int64_t ldx, int32_t part, void *stream) {
    DeviceGuard dg_(h);
    if (nrhs < 0 || (nrhs > 0 && ldx < h->n) || part < 0 || part > 2) {
        glu::set_error("bad multi-RHS solve arguments");
        return GLU_EINVAL;
    }
    if (nrhs == 0) return GLU_OK;
    cudaStream_t s = (cudaStream_t)stream;
    i64 rc;
    if (part != 1 && (rc = check_zero_pivot(h, lu, s)) != GLU_OK) return rc;
    if ((rc = run_solves(h, lu, x, (int)part, s, (int)nrhs, ldx)) != GLU_OK) return rc;
    GLU_CUDA(cudaStreamSynchronize(s));
    return GLU_OK;
}

// Batch solves: set b's factors at lu + b * lu_stride,
// its right-hand side / solution at x + b * ldx; one pair of dataflow
// launches for all sets.  status[b] = -1, or the zero-diagonal column the
// reference's upper_solve raises for that set (its x is then unspecified).
extern "C" int64_t glu_solve_batch_device(glu_handle *h, const double *lu, int64_t lu_stride, double *x,
                                          int64_t nb, int64_t ldx, int64_t *status, void *stream) {
    DeviceGuard dg_(h);
    if (nb < 0 || (nb > 0 && (ldx < h->n || lu_stride < h->nnz))) {
        glu::set_error("bad batch solve arguments");
        return GLU_EINVAL;
    }
    if (nb == 0) return GLU_OK;
    cudaStream_t s = (cudaStream_t)stream;
    int *dfail = nullptr;
    GLU_CUDA(cudaMallocAsync((void **)&dfail, sizeof(int) * nb, s));
    GLU_CUDA(cudaMemsetAsync(dfail, 0xff, sizeof(int) * nb, s));  // -1
    zero_pivot_batch_kernel<<<h->sm_count * 4, 256, 0, s>>>(lu, lu_stride, h->diag_pos, (i32)h->n,
                                                           (int)nb, dfail);
    GLU_CUDA(cudaGetLastError());
    i64 rc = run_solves(h, lu, x, 0, s, (int)nb, ldx, lu_stride);
    std::vector<int> f((size_t)nb, -1);
    cudaMemcpyAsync(f.data(), dfail, sizeof(int) * nb, cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(dfail, s);
    GLU_CUDA(cudaStreamSynchronize(s));
    if (rc != GLU_OK) return rc;
    for (i64 b = 0; b < nb; b++) status[b] = f[b];
    return GLU_OK;
}

extern "C" int64_t glu_factor_host(glu_handle *h, const double *a_vals, double *lu_out, double thresh) {
    DeviceGuard dg_(h);
    if (h->nz < 0) { glu::set_error("glu_set_input_pattern not called"); return GLU_EINVAL; }
    i64 rc = ensure_staging(h);
    if (rc != GLU_OK) return rc;
    cudaStream_t s = h->stream;
    GLU_CUDA(cudaMemcpyAsync(h->d_a, a_vals, sizeof(double) * h->nz, cudaMemcpyHostToDevice, s));
    if ((rc = glu_scatter_device(h, h->d_a, h->d_v, s)) != GLU_OK) return rc;
    const bool split = h->tail_t0 < h->n && h->tail_t0 > 0;
    if (split && !h->ev_main) {
        GLU_CUDA(cudaEventCreateWithFlags(&h->ev_main, cudaEventDisableTiming));
        GLU_CUDA(cudaEventCreateWithFlags(&h->ev_copy, cudaEventDisableTiming));
        GLU_CUDA(cudaStreamCreateWithFlags(&h->stream2, cudaStreamNonBlocking));
    }
    if ((rc = launch_factor(h, h->d_v, thresh, s)) != GLU_OK) return rc;
    if (h->sn) {
        // the supernodal engine's panels become final one by one: their
        // values travel to the host while the kernel still runs
        if ((rc = glu::sn_copy_out(h->sn, h->d_v, lu_out, s)) != GLU_OK) return rc;
    } else if (split) {
        // the columns below the dense tail are final when the main kernel
        // ends: copy them out while the cluster tail kernel runs
        const i64 head = h->col_ptr_h_t0;
        GLU_CUDA(cudaStreamWaitEvent(h->stream2, h->ev_main, 0));
        GLU_CUDA(cudaMemcpyAsync(lu_out, h->d_v, sizeof(double) * head, cudaMemcpyDeviceToHost, h->stream2));
        GLU_CUDA(cudaEventRecord(h->ev_copy, h->stream2));
        GLU_CUDA(cudaMemcpyAsync(lu_out + head, h->d_v + head, sizeof(double) * (h->nnz - head),
                                 cudaMemcpyDeviceToHost, s));
        GLU_CUDA(cudaStreamWaitEvent(s, h->ev_copy, 0));
    } else {
        GLU_CUDA(cudaMemcpyAsync(lu_out, h->d_v, sizeof(double) * h->nnz, cudaMemcpyDeviceToHost, s));
    }
    return read_fail(h, s);
}

extern "C" int64_t glu_solve_host(glu_handle *h, const double *lu, const double *b, double *x) {
    DeviceGuard dg_(h);
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
