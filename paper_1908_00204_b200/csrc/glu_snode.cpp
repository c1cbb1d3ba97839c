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
//   * pushes into a target panel K are applied in ascending source panel,
//     one per stage (stage(P,K) = max(stage(P factored), previous push + 1));
//   * inside a push, every target receives the panel's columns in ascending
//     order (the kernel's chains), and panel K is factored in the stage after
//     its last push.
//
// Each stage has two phases (the kernel's only synchronisation):
//   0  TRSM(P,c)  rows below the panel, 32 at a time: divide and in-panel
//                 updates (factoring the w x w diagonal block locally)
//      TRI(push)  U(P, K) = forward substitution inside the source panel
//   1  RECT(push,c) rows below P, 32 at a time, into every column of K
//      DIAG(P)    the factored diagonal block written back
// Empty phases are dropped.
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
    std::vector<i32> fstage(np, 0), seen(np, -1), push_stage;
    std::vector<char> push_tri;
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
        i64 last = -1;
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
            last = std::max<i64>(fstage[p], last + 1);
            P->push.push_back(I4{p, (i32)r0, (i32)r1, (i32)K});
            push_stage.push_back((i32)last);
            push_tri.push_back(tri > 0);
        }
        fstage[K] = (i32)(last + 1);
    }
    // in-panel MACs (DIAG + TRSM): every source j of a column c inside its panel
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

    // 6. tasks in phase order: two phases per stage, empty phases dropped.
    //   phase 2s     TRSM(P) of the panels factored in stage s and TRI of the
    //                stage's pushes; both factor P's w x w diagonal block
    //                themselves when it is not yet factored (kSnLocal: the
    //                panel's own stage), from values no task of the phase writes
    //   phase 2s + 1 RECT of the stage's pushes, and DIAG(P), which writes
    //                the factored block back (nothing in this phase reads it)
    // Inside a phase tasks are ordered by estimated cost, largest first, so
    // the static round-robin deal gives every warp a similar load.
    i64 n_stages = 0;
    for (i64 p = 0; p < np; p++) n_stages = std::max<i64>(n_stages, fstage[p] + 1);
    for (i32 s : push_stage) n_stages = std::max<i64>(n_stages, s + 1);
    P->n_stages = n_stages;
    const i64 nph = 2 * n_stages;
    auto chunks = [](i64 h) { return (h + 31) / 32; };
    struct T {
        i64 cost;
        i32 f, pi, chunk, kind, r0, r1;
    };
    std::vector<T> all;
    const i64 npush = (i64)P->push.size();
    constexpr i64 kTaskCost = 4000;  // ~1 us of latency, in MACs
    for (i64 p = 0; p < np; p++) {
        const I4 pn = P->pan[p];
        const i64 w = pn.y - pn.x;
        all.push_back({kTaskCost + w * w * w / 3, 2 * fstage[p] + 1, (i32)p, 0, kSnDiag, 0, 0});
        for (i64 c = 0; c < chunks(pn.w); c++) {
            const i64 rows = std::min<i64>(32, pn.w - 32 * c);
            all.push_back({kTaskCost + w * w * w / 3 + rows * w * w / 2, 2 * fstage[p], (i32)p, (i32)c,
                           kSnTrsm | kSnLocal, 0, 0});
        }
    }
    for (i64 x = 0; x < npush; x++) {
        const I4 ps = P->push[x];
        const I4 pn = P->pan[ps.x];
        const i64 w = pn.y - pn.x, np_ = ps.z - ps.y;
        const bool local = push_stage[x] == fstage[ps.x];
        if (push_tri[x])
            all.push_back({kTaskCost + np_ * w * w / 2 + (local ? w * w * w / 3 : 0), 2 * push_stage[x], ps.x, 0,
                           kSnTri | (local ? kSnLocal : 0), ps.y, ps.z});
        for (i64 c = 0; c < chunks(pn.w); c++) {
            const i64 rows = std::min<i64>(32, pn.w - 32 * c);
            all.push_back({kTaskCost + rows * np_ * w, 2 * push_stage[x] + 1, ps.x, (i32)c, kSnRect, ps.y, ps.z});
        }
    }
    std::stable_sort(all.begin(), all.end(), [](const T &a, const T &b) {
        return a.f != b.f ? a.f < b.f : a.cost > b.cost;
    });
    if ((i64)all.size() >= (i64)INT32_MAX) {
        set_error("supernodal plan: >= 2^31 tasks");
        return GLU_EINVAL;
    }
    std::vector<i32> remap(nph, -1);
    i64 live = 0;
    for (const T &t : all)
        if (remap[t.f] < 0) remap[t.f] = (i32)live++;
    P->phase_ptr.assign(live + 1, 0);
    for (const T &t : all) P->phase_ptr[remap[t.f] + 1]++;
    for (i64 f = 0; f < live; f++) P->phase_ptr[f + 1] += P->phase_ptr[f];
    // two records per task: {kind << 28 | chunk, phase, p0, p1}, {s1, rows below p1, pair0, pair1}
    P->tasks.resize(2 * all.size());
    for (size_t i = 0; i < all.size(); i++) {
        const T &t = all[i];
        const I4 pn = P->pan[t.pi];
        P->tasks[2 * i] = I4{(t.kind << 27) | t.chunk, remap[t.f], pn.x, pn.y};
        P->tasks[2 * i + 1] = I4{(i32)s1_of(pn.z), pn.w, t.r0, t.r1};
    }
    return GLU_OK;
}

}  // namespace glu
