// glu_snode.cpp -- host plan of the supernodal engine (glu_snode.cu).
//
// The per-MAC plan of glu_host.cpp costs ~3 B per MAC: 125 GB for the
// G3-like cfg4 (3.8e10 MACs).  This plan indexes the same MACs by blocks:
//
//   supernode S = [s0, s1)   fundamental: L(:,c-1) = {c} u L(:,c) and
//                            U(c-1,c) != 0, so every column of S has the rows
//                            (c, s1) u R_S below its diagonal (R_S: rows
//                            below the supernode, shared)
//   panel P = [p0, p1)       <= kSnW consecutive columns of one supernode
//   pair (S, k)              target column k of S (U(s1-1,k) != 0).  The
//                            rows of S present in column k are a suffix
//                            [a_k, s1) stored contiguously (fill: L(r,j) != 0
//                            for j < r in S, so U(j,k) != 0 implies U(r,k)),
//                            and R_S sits in column k at relmap positions
//                            (|R_S| int32 per pair -- 0.1 B per MAC on cfg4)
//   push (P, K)              the MACs of panel P's sources into target panel K
//
// Every MAC of the reference is A_s(r,k) -= L(r,j) * U(j,k) for a source
// column j with U(j,k) != 0 and r in L(:,j) (levlu/_kernels.py:57-59); this
// plan covers exactly those MACs (source j in [max(a_k, p0), p1) of every
// push into column k), and orders them per target in ascending j (contract
// A, the left-looking order, _kernels.py:37-76):
//
//   * pushes into a target panel K are applied one after another in
//     ascending source panel (a counter per target panel), and panel K is
//     factored after its last push;
//   * inside a push, every target receives the panel's columns in ascending
//     order (the kernel's chains).
//
// The kernel is a dataflow walk over five task kinds (no phases, no grid
// barrier; step 6 below has the counters):
//   TRSM(P,c)   32 rows below panel P: factor the w x w diagonal block
//               locally, divide, in-panel updates (chunk 0 also stores the
//               factored block in a scratch area)
//   WB(P)       the factored block written back in place once every TRSM
//               chunk of P has read the unfactored one
//   RECT(x,c)   push x = (P, K), 32 rows below P into every column of K,
//               after the forward substitution U(P, K) inside P's block
//   UW(x)       writes the solved U(P, K) when several RECT chunks read it
//   RG          a run of pushes from one-column panels into one target
//               panel, applied by one warp on a shared-memory image
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "glu_b200.h"
#include "glu_internal.h"

using i64 = int64_t;
using i32 = int32_t;

namespace glu {

namespace {

template <class F>
void parallel_for(i64 count, int nt, i64 block, F fn) {
    std::atomic<i64> next{0};
    auto work = [&](int tid) {
        while (true) {
            const i64 b = next.fetch_add(block);
            if (b >= count) break;
            fn(tid, b, std::min<i64>(count, b + block));
        }
    };
    std::vector<std::thread> th;
    for (int t = 1; t < nt; t++) th.emplace_back(work, t);
    work(0);
    for (auto &t : th) t.join();
}

}  // namespace

int64_t sn_build(int64_t n, const int64_t *col_ptr, const int64_t *row_idx, const int64_t *diag_pos,
                 const int64_t *row_ptr, const int64_t *col_idx, const int64_t *csc_pos, int n_threads,
                 SnPlan *P) {
    (void)csc_pos;
    if (col_ptr[n] >= (int64_t)INT32_MAX) {
        set_error("pattern has >= 2^31 entries; slot indices are int32 on the device");
        return GLU_EINVAL;
    }
    const int nt = n_threads > 0 ? n_threads : (int)std::max(1u, std::thread::hardware_concurrency());
    P->n = n;
    P->nnz = col_ptr[n];
    P->col_ptr_h.assign(col_ptr, col_ptr + n + 1);
    auto llen = [&](i64 c) { return col_ptr[c + 1] - diag_pos[c] - 1; };

    // 1. fundamental supernodes
    std::vector<i32> sn_of(n);
    std::vector<i64> s0v;
    for (i64 c = 0; c < n; c++) {
        const bool join = c > 0 && llen(c - 1) == llen(c) + 1 && row_idx[diag_pos[c - 1] + 1] == c &&
                          diag_pos[c] > col_ptr[c] && row_idx[diag_pos[c] - 1] == c - 1;
        if (!join) s0v.push_back(c);
        sn_of[c] = (i32)s0v.size() - 1;
    }
    const i64 ns = (i64)s0v.size();
    s0v.push_back(n);
    auto s1_of = [&](i64 S) { return s0v[S + 1]; };

    // 2. panels of <= kSnW columns, as even as possible inside a supernode
    std::vector<i32> pan_of(n);
    std::vector<i64> pan0;
    std::vector<i32> pan_sn;
    for (i64 S = 0; S < ns; S++) {
        const i64 s0 = s0v[S], w = s1_of(S) - s0, m = (w + kSnW - 1) / kSnW;
        for (i64 t = 0; t < m; t++) {
            const i64 a = s0 + (w * t) / m, b = s0 + (w * (t + 1)) / m;
            for (i64 c = a; c < b; c++) pan_of[c] = (i32)pan0.size();
            pan0.push_back(a);
            pan_sn.push_back((i32)S);
        }
    }
    const i64 np = (i64)pan0.size();
    pan0.push_back(n);

    // 3. (S, k) pairs: inside targets (s0, s1), then row s1-1's U columns
    std::vector<i64> pair_ptr(ns + 1, 0), map_ptr(ns + 1, 0);
    std::vector<i64> nR(ns);
    for (i64 S = 0; S < ns; S++) {
        const i64 last = s1_of(S) - 1;
        nR[S] = llen(last);
        i64 nout = 0;
        for (i64 t = row_ptr[last + 1] - 1; t >= row_ptr[last] && col_idx[t] > last; t--) nout++;
        pair_ptr[S + 1] = pair_ptr[S] + (s1_of(S) - s0v[S] - 1) + nout;
        map_ptr[S + 1] = map_ptr[S] + nout * nR[S];
    }
    if (pair_ptr[ns] >= (i64)INT32_MAX || map_ptr[ns] >= (i64)INT32_MAX) {
        set_error("supernodal plan: >= 2^31 pairs or map entries");
        return GLU_EINVAL;
    }
    P->pairs.assign(pair_ptr[ns], I4{0, 0, 0, 0});
    P->col_a.resize(n);
    for (i64 S = 0; S < ns; S++) P->col_a[s0v[S]] = (i32)s0v[S];
    P->relmap.assign(map_ptr[ns], -1);
    std::atomic<i64> bad{-1};
    auto mark_bad = [&](i64 k) {
        i64 cur = bad.load();
        while ((cur < 0 || k < cur) && !bad.compare_exchange_weak(cur, k)) {}
    };
    parallel_for(ns, nt, 256, [&](int, i64 b, i64 e) {
        for (i64 S = b; S < e; S++) {
            const i64 s0 = s0v[S], s1 = s1_of(S), last = s1 - 1;
            i64 q = pair_ptr[S];
            for (i64 k = s0 + 1; k < s1; k++) {  // inside: suffix [k - u, k) of U rows
                i64 u = 0;
                while (diag_pos[k] - 1 - u >= col_ptr[k] && row_idx[diag_pos[k] - 1 - u] >= s0) u++;
                if (u == 0 || row_idx[diag_pos[k] - u] != k - u) { mark_bad(k); continue; }
                P->pairs[q++] = I4{(i32)k, (i32)(k - u), (i32)(diag_pos[k] + (s1 - k)), -1};
                P->col_a[k] = (i32)(k - u);
            }
            i64 t0 = row_ptr[last + 1];
            while (t0 > row_ptr[last] && col_idx[t0 - 1] > last) t0--;
            i64 mo = map_ptr[S];
            for (i64 t = t0; t < row_ptr[last + 1]; t++, q++) {
                const i64 k = col_idx[t];
                const int64_t *rb = row_idx + col_ptr[k], *re = row_idx + diag_pos[k];
                const i64 pos = (i64)(std::lower_bound(rb, re, (int64_t)s0) - row_idx);
                const i64 a = row_idx[pos];
                if (pos >= diag_pos[k] || a >= s1 || pos + (s1 - 1 - a) >= diag_pos[k] ||
                    row_idx[pos + (s1 - 1 - a)] != s1 - 1) {
                    mark_bad(k);
                    continue;
                }
                P->pairs[q] = I4{(i32)k, (i32)a, (i32)(pos + (s1 - a)), nR[S] > 0 ? (i32)mo : -1};
                mo += nR[S];
            }
        }
    });
    if (bad.load() >= 0) {
        set_error("supernodal plan: column " + std::to_string(bad.load()) +
                  " lacks a fill-in slot (pattern not closed under elimination)");
        return GLU_MISMATCH;
    }

    // 4. relmap: R_S's rows located in every outside target column
    std::vector<std::vector<i32>> posmaps(nt);
    parallel_for(n, nt, 512, [&](int tid, i64 b, i64 e) {
        std::vector<i32> &pm = posmaps[tid];
        if (pm.empty()) pm.assign(n, -1);
        for (i64 k = b; k < e; k++) {
            const i64 cb = col_ptr[k], ce = col_ptr[k + 1];
            bool any = false;
            for (i64 m = cb; m < diag_pos[k]; m++) {
                const i64 S = sn_of[row_idx[m]];
                if (m > cb && sn_of[row_idx[m - 1]] == S) continue;
                if (s1_of(S) > k || nR[S] == 0) continue;
                if (!any) {
                    for (i64 p = cb; p < ce; p++) pm[row_idx[p]] = (i32)p;
                    any = true;
                }
                const I4 *pb = P->pairs.data() + pair_ptr[S], *pe = P->pairs.data() + pair_ptr[S + 1];
                const I4 *it = std::lower_bound(pb, pe, (i32)k, [](const I4 &x, i32 v) { return x.x < v; });
                if (it == pe || it->x != (i32)k) { mark_bad(k); continue; }
                const i64 last = s1_of(S) - 1;
                for (i64 i = 0; i < nR[S]; i++) {
                    const i32 pos = pm[row_idx[diag_pos[last] + 1 + i]];
                    if (pos < 0) { mark_bad(k); break; }
                    P->relmap[it->w + i] = pos;
                }
            }
            if (any)
                for (i64 p = cb; p < ce; p++) pm[row_idx[p]] = -1;
        }
    });
    posmaps.clear();
    if (bad.load() >= 0) {
        set_error("supernodal plan: column " + std::to_string(bad.load()) +
                  " lacks a fill-in slot (pattern not closed under elimination)");
        return GLU_MISMATCH;
    }

    // 5. pushes and stages (target panels in ascending order)
    P->sn.resize(ns);
    for (i64 S = 0; S < ns; S++)
        P->sn[S] = I4{(i32)s0v[S], (i32)s1_of(S), (i32)nR[S], (i32)pair_ptr[S]};
    P->pan.resize(np);
    for (i64 p = 0; p < np; p++) {
        const i64 S = pan_sn[p];
        P->pan[p] = I4{(i32)pan0[p], (i32)pan0[p + 1], (i32)S, (i32)((s1_of(S) - pan0[p + 1]) + nR[S])};
    }
    std::vector<i32> seen(np, -1);
    std::vector<char> push_tri;
    std::vector<i64> push_macs;
    std::vector<i32> srcs;
    i64 macs = 0;
    for (i64 K = 0; K < np; K++) {
        const i64 k0 = pan0[K], k1 = pan0[K + 1];
        srcs.clear();
        for (i64 k = k0; k < k1; k++) {
            for (i64 m = col_ptr[k]; m < diag_pos[k]; m++) {
                const i64 j = row_idx[m];
                if (j >= k0) break;
                const i64 S = sn_of[j];
                if (m > col_ptr[k] && sn_of[row_idx[m - 1]] == S) continue;
                const i64 hi = std::min<i64>(s1_of(S), k0);
                for (i64 p = pan_of[j]; p <= pan_of[hi - 1]; p++)
                    if (seen[p] != (i32)K) { seen[p] = (i32)K; srcs.push_back((i32)p); }
            }
        }
        std::sort(srcs.begin(), srcs.end());
        for (i32 p : srcs) {
            const I4 pn = P->pan[p];
            const i64 S = pn.z, s1 = s1_of(S);
            const I4 *pb = P->pairs.data() + pair_ptr[S], *pe = P->pairs.data() + pair_ptr[S + 1];
            auto lb = [](const I4 &x, i32 v) { return x.x < v; };
            const i64 r0 = std::lower_bound(pb, pe, (i32)k0, lb) - P->pairs.data();
            const i64 r1 = std::lower_bound(pb, pe, (i32)k1, lb) - P->pairs.data();
            i64 pm = 0, tri = 0;
            for (i64 q = r0; q < r1; q++) {
                const i64 a = P->pairs[q].y;
                if (a >= pn.y) continue;
                for (i64 j = std::max<i64>(a, pn.x); j < pn.y; j++) {
                    pm += (s1 - 1 - j) + nR[S];
                    tri += pn.y - 1 - j;
                }
            }
            if (pm == 0) continue;
            macs += pm;
            P->push.push_back(I4{p, (i32)r0, (i32)r1, (i32)K});
            push_tri.push_back(tri > 0);
            push_macs.push_back(pm);
        }
    }
    // in-panel MACs (TRSM's diagonal-block factorization and row updates)
    for (i64 p = 0; p < np; p++) {
        const I4 pn = P->pan[p];
        const i64 S = pn.z, s1 = s1_of(S);
        for (i64 c = pn.x + 1; c < pn.y; c++) {
            i64 a = c;
            while (a - 1 >= pn.x && diag_pos[c] - (c - (a - 1)) >= col_ptr[c] &&
                   row_idx[diag_pos[c] - (c - (a - 1))] == a - 1)
                a--;
            for (i64 j = a; j < c; j++) macs += (s1 - 1 - j) + nR[S];
        }
    }
    P->macs = macs;

    // 6. dataflow tasks.  Per panel P: nch = max(1, ceil(rows below / 32))
    // TRSM chunks; per push x = (P, K): nch(P) RECT chunks (rows below P,
    // 32 each; the forward substitution for U(P, K) folded in) and, when
    // U(P, K) changes and several chunks read it, one U-writer.  Counters:
    //   in[K]  RECT chunks of pushes into K done; push x waits for
    //          in[K] >= need(x) (every earlier push into K), TRSM(K) for
    //          in[K] >= total_in(K)
    //   f[P]   TRSM chunks of P done; RECT(x) waits for f[P] >= nch(P)
    //   U-writer of x waits for in[K] >= need(x) + nch(P)
    // A run of consecutive one-chunk pushes from one-column panels into K
    // (most pushes of a nested-dissection order: the small separators'
    // columns) is one RG task instead: a warp applies them in order, waiting
    // for each source panel's TRSM as it goes, and counts them all at the
    // end -- the chain of pushes into K then costs an L2 round trip per push
    // instead of a cross-SM hand-off.
    // Tasks are ordered by their start in an as-soon-as-possible schedule
    // under a latency model (hop + per-task cost); every dependency starts
    // strictly earlier, so the order is topological and the kernel's static
    // deal (each warp walks its tasks in order) cannot deadlock.
    const i64 npush = (i64)P->push.size();
    auto chunks = [](i64 h) { return std::max<i64>(1, (h + 31) / 32); };
    P->panm.assign(np, I4{0, 0, -1, 0});  // .w: completions (WB, UWs) that finish the panel's values
    i64 dbl = 0;
    for (i64 p = 0; p < np; p++) {
        const I4 pn = P->pan[p];
        const i64 w = pn.y - pn.x;
        P->panm[p].y = (i32)chunks(pn.w);
        if (w >= 2) {
            P->panm[p].z = (i32)dbl;
            dbl += w * w;
        }
    }
    if (dbl >= (i64)INT32_MAX) {
        set_error("supernodal plan: diagonal-block scratch >= 2^31 doubles");
        return GLU_EINVAL;
    }
    P->n_dblk = dbl;
    // latency model (us), calibrated on the B200 traces (tools/sn_critpath.py)
    // (GLU_SN_HOP: tuning override of the hand-off latency, order only)
    const double kHop = std::getenv("GLU_SN_HOP") ? std::max(0.1, std::atof(std::getenv("GLU_SN_HOP"))) : 2.5;  // release -> observe
    constexpr double kMacsPerUs = 4000.0;        // one warp's FP64 chain rate
    constexpr double kGatherSrcUs = 0.15;        // one push inside an RG (shared-memory chains)
    constexpr double kGatherUs = 3.0;            // an RG's staging loads
    constexpr i64 kMaxGather = kRgPushes;        // pushes per RG task (one per lane)
    // runs shorter than this stay RECT tasks; 1 (every eligible run an RG task) measured best:
    // cfg4 48.5 vs 48.8 ms (3), g400 7.54 vs 7.74, g800 19.8 vs 20.3 (GLU_SN_MINGATHER: tuning override)
    const i64 kMinGather = std::getenv("GLU_SN_MINGATHER") ? std::max<i64>(1, std::atoll(std::getenv("GLU_SN_MINGATHER"))) : 1;
    std::vector<double> f_done(np, 0.0), f_start(np, 0.0);
    struct T {
        double start, cost;
        i32 kind, pi, chunk, x;
    };
    std::vector<T> all;
    all.reserve((size_t)(np + 2 * npush));
    double crit = 0.0;
    // RG slot bookkeeping: the slots an RG touches all lie in its target
    // panel's columns; mark[slot - col_ptr[k0]] = (generation, index in T)
    i64 max_span = 0;
    for (i64 K = 0; K < np; K++) max_span = std::max<i64>(max_span, col_ptr[pan0[K + 1]] - col_ptr[pan0[K]]);
    std::vector<i32> mark_gen((size_t)max_span, -1), mark_idx((size_t)max_span, 0);
    i32 gen = -1;
    std::vector<i32> cur_slots;
    i64 x = 0;
    for (i64 K = 0; K < np; K++) {
        double t = 0.0;
        i64 need = 0;
        const i64 kbase = col_ptr[pan0[K]];
        // RG: a run of consecutive one-chunk pushes from one-column panels
        // into K, applied by one warp in order (no hand-off between them)
        i64 g_first = -1, g_cnt = 0;
        double g_key = 0.0, g_cost = 0.0, g_t0 = 0.0;
        size_t g_idx0 = 0, g_uidx0 = 0;
        i64 g_rows = 0, g_chunks = 0;  // the open RG's L rows and RECT chunks
        auto slot_of = [&](const I4 &pr, i64 tr) -> i64 {  // row tr below a one-column source, pair pr
            return pr.w >= 0 ? (i64)P->relmap[pr.w + tr] : (i64)pr.z + tr;
        };
        auto close_g = [&]() {
            if (g_cnt >= kMinGather) {
                const i32 r = (i32)P->rg.size();
                P->rg.push_back(I4{(i32)P->rg_slot.size(), (i32)cur_slots.size(), (i32)g_idx0, (i32)g_uidx0});
                P->rg_slot.insert(P->rg_slot.end(), cur_slots.begin(), cur_slots.end());
                P->rg_chunks.push_back((i32)g_chunks);
                all.push_back({g_key, g_cost, kSnRg << 2, r, (i32)g_cnt, (i32)g_first});
            } else if (g_cnt > 0) {
                // too short: one RECT task per push, chained as usual
                P->rg_idx.resize(g_idx0);
                P->rg_uidx.resize(g_uidx0);
                double tt = g_t0;
                for (i64 y = g_first; y < g_first + g_cnt; y++) {
                    const i32 src = P->push[y].x;
                    const i64 nch = chunks(P->pan[src].w);
                    const double st = std::max(tt, f_done[src]) + kHop;
                    const double per = 2.5 + (double)push_macs[y] / (double)nch / kMacsPerUs;
                    for (i64 c = 0; c < nch; c++) all.push_back({st, per, kSnRect << 2, src, (i32)c, (i32)y});
                    tt = st + per;
                }
                t = std::max(t, tt);
            }
            g_cnt = 0;
        };
        for (; x < npush && P->push[x].w == (i32)K; x++) {
            const I4 ps = P->push[x];
            const I4 pn = P->pan[ps.x];
            const i64 w = pn.y - pn.x, npair = ps.z - ps.y, nc = chunks(pn.w);
            P->push_need.push_back((i32)need);
            const i64 hh = pn.w;
            if (w == 1 && hh <= kRgRows / 4 && npair * hh <= kRgIdx && npair * (hh + 1) <= kRgSlots) {
                const double ready = f_done[ps.x];
                const i64 h = hh;
                // new distinct slots (targets and U(p0, k)) this push would add to the
                // open RG, and its MAC indices (pair q, row tr at q * h + tr)
                i64 fresh = 0;
                if (g_cnt > 0)
                    for (i64 q = ps.y; q < ps.z; q++) {
                        const I4 pr = P->pairs[q];
                        if (pr.y >= pn.y) continue;
                        if (mark_gen[(i64)pr.z - 1 - kbase] != gen) fresh++;
                        for (i64 tr = 0; tr < h; tr++)
                            if (mark_gen[slot_of(pr, tr) - kbase] != gen) fresh++;
                    }
                // (a late source does not split the run: the pushes into K run in
                // order anyway, so the ones after it wait for it either way)
                if (!(g_cnt > 0 && g_cnt < kMaxGather && g_rows + h <= kRgRows &&
                      (i64)cur_slots.size() + fresh <= kRgSlots &&
                      (i64)(P->rg_idx.size() - g_idx0) + npair * h <= kRgIdx &&
                      (i64)(P->rg_uidx.size() - g_uidx0) + npair <= kRgPushes * kSnW)) {
                    close_g();
                    g_first = x;
                    g_t0 = t;
                    t = std::max(t, ready) + kHop + kGatherUs;
                    g_key = t - kGatherUs;
                    g_cost = kGatherUs;
                    gen++;
                    cur_slots.clear();
                    g_idx0 = P->rg_idx.size();
                    g_uidx0 = P->rg_uidx.size();
                    g_rows = g_chunks = 0;
                }
                // the push's MACs as indices into the RG's slot list (pair q, row tr
                // at q * h + tr), and per pair the index of U(p0, k)
                auto index_of = [&](i64 slot) -> uint16_t {
                    const i64 sl = slot - kbase;
                    if (mark_gen[sl] != gen) {
                        mark_gen[sl] = gen;
                        mark_idx[sl] = (i32)cur_slots.size();
                        cur_slots.push_back((i32)slot);
                    }
                    return (uint16_t)mark_idx[sl];
                };
                for (i64 q = ps.y; q < ps.z; q++) {
                    const I4 pr = P->pairs[q];
                    const bool ok = pr.y < pn.y;
                    P->rg_uidx.push_back(ok ? index_of((i64)pr.z - 1) : (uint16_t)0);
                    for (i64 tr = 0; tr < h; tr++) P->rg_idx.push_back(ok ? index_of(slot_of(pr, tr)) : (uint16_t)0);
                }
                // after its sources' TRSM tasks in the list (topological order)
                g_key = std::max(g_key, f_start[ps.x] + 1e-3);
                t = std::max(t, ready) + kGatherSrcUs;
                g_cost += kGatherSrcUs;
                g_cnt++;
                g_rows += h;
                g_chunks += nc;
                need += nc;
                continue;
            }
            close_g();
            const double st = std::max(t, f_done[ps.x]) + kHop;
            const double per = 2.5 + (double)push_macs[x] / (double)nc / kMacsPerUs +
                               (push_tri[x] ? 0.05 * (double)(w * w) : 0.0);
            const bool uw = push_tri[x] && nc > 1;
            const i32 flags = (push_tri[x] ? kSnTriF : 0) | (push_tri[x] && !uw ? kSnWriteU : 0);
            for (i64 c = 0; c < nc; c++) all.push_back({st, per, (kSnRect << 2) | flags, (i32)ps.x, (i32)c, (i32)x});
            t = st + per;
            if (uw) {
                all.push_back({t + kHop, 1.0 + 0.05 * (double)(w * w * npair) / 16.0, kSnUw << 2,
                               (i32)ps.x, 0, (i32)x});
                P->panm[K].w++;  // the UW writes into K's columns: K is final after it
            }
            need += nc;
        }
        close_g();
        P->panm[K].x = (i32)need;
        const I4 pn = P->pan[K];
        const i64 w = pn.y - pn.x, nc = chunks(pn.w);
        const double st = (need > 0 ? t + kHop : 0.0);
        const double cost = 0.5 + 1.2 * (double)w + (double)(32 * w * w / 2) / kMacsPerUs;
        for (i64 c = 0; c < nc; c++) all.push_back({st, cost, kSnTrsm << 2, (i32)K, (i32)c, -1});
        if (w >= 2) {  // WB: the factored block back in place once every TRSM chunk has read it
            all.push_back({st + cost + kHop, 0.5, kSnWb << 2, (i32)K, 0, -1});
            P->panm[K].w++;
        }
        f_start[K] = st;
        f_done[K] = st + cost;
        crit = std::max(crit, f_done[K]);
    }
    if ((i64)P->rg_idx.size() >= (i64)INT32_MAX || (i64)P->rg_slot.size() >= (i64)INT32_MAX) {
        set_error("supernodal plan: RG index arrays >= 2^31 entries");
        return GLU_EINVAL;
    }
    std::stable_sort(all.begin(), all.end(), [](const T &a, const T &b) {
        return a.start != b.start ? a.start < b.start : a.cost > b.cost;
    });
    if ((i64)all.size() >= (i64)INT32_MAX) {
        set_error("supernodal plan: >= 2^31 tasks");
        return GLU_EINVAL;
    }
    P->crit_ns = (i64)(crit * 1e3);
    // three records per task (glu_internal.h SnPlan::tasks)
    P->tasks.resize(3 * all.size());
    P->task_cost.resize(all.size());
    for (size_t i = 0; i < all.size(); i++) P->task_cost[i] = (float)all[i].cost;
    parallel_for((i64)all.size(), nt, 1 << 16, [&](int, i64 b, i64 e) {
        for (i64 i = b; i < e; i++) {
            const T &t = all[i];
            if (t.kind == (kSnRg << 2)) {
                // {code << 27 | pushes, first MAC index, first U index, RECT chunks}, {first slot, slots,
                // first push, pushes}, {K, need, 0, 0}
                const I4 g = P->rg[t.pi];
                const I4 ps = P->push[t.x];
                P->tasks[3 * i] = I4{(i32)((uint32_t)t.kind << 27 | (uint32_t)t.chunk), g.z, g.w, P->rg_chunks[t.pi]};
                P->tasks[3 * i + 1] = I4{g.x, g.y, t.x, t.chunk};
                P->tasks[3 * i + 2] = I4{ps.w, P->push_need[t.x], 0, 0};
                continue;
            }
            const I4 pn = P->pan[t.pi];
            I4 c{0, 0, 0, 0};
            i32 pr0 = 0, pr1 = 0;
            if (t.x >= 0) {
                const I4 ps = P->push[t.x];
                pr0 = ps.y;
                pr1 = ps.z;
                c = I4{ps.w, P->push_need[t.x], 0, 0};
            }

            P->tasks[3 * i] = I4{(i32)((uint32_t)t.kind << 27 | (uint32_t)t.chunk), t.pi, pn.x, pn.y};
            P->tasks[3 * i + 1] = I4{(i32)s1_of(pn.z), pn.w, pr0, pr1};
            P->tasks[3 * i + 2] = c;
        }
    });
    return GLU_OK;
}

}  // namespace glu
