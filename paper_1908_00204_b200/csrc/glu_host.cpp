// glu_host.cpp -- host side of the B200 GLU3.0 path: symbolic fill-in,
// relaxed dependency detection, levelization, and the precomputed
// destination-owned update plan that the persistent sm_100a kernel walks.
//
// Everything here runs once per sparsity pattern.  The pattern, the
// dependency lists and the levels are uniquely determined by the input
// pattern, so any correct algorithm reproduces the reference's arrays
// bit for bit; parity is checked against the reference's own outputs in
// tests/test_analysis.py.
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "glu_b200.h"
#include "glu_internal.h"

namespace glu {

thread_local std::string g_last_error;

void set_error(const std::string &s) { g_last_error = s; }

}  // namespace glu

using glu::set_error;
using i64 = int64_t;
using i32 = int32_t;

extern "C" int64_t glu_last_error(char *buf, int64_t len) {
    const std::string &e = glu::g_last_error;
    if (buf && len > 0) {
        size_t m = std::min<size_t>((size_t)len - 1, e.size());
        std::memcpy(buf, e.data(), m);
        buf[m] = 0;
    }
    return (int64_t)e.size();
}

// ---------------------------------------------------------------------------
// Symbolic fill-in (symbolic.py:92-145).  Column j's filled pattern is the
// set of rows reachable from A(:,j) through the L columns left of j.  We use
// the Gilbert-Peierls DFS of symbolic.py:66-89 plus Eisenstat-Liu symmetric
// pruning: once column s is known, any column k < s with both L(s,k) and
// U(k,s) nonzero only needs its L rows <= s for later reachability (rows
// below s of L(:,k) are contained in L(:,s)).  Pruning changes the
// traversal cost only, never the reach set.
// ---------------------------------------------------------------------------
struct glu_pattern {
    i64 n = 0;
    std::vector<i64> col_ptr, row_idx, diag_pos, row_ptr, col_idx, csc_pos;
};

static void build_csr(i64 n, const i64 *col_ptr, const i64 *row_idx, i64 *row_ptr, i64 *col_idx,
                      i64 *csc_pos) {
    i64 nnz = col_ptr[n];
    std::fill(row_ptr, row_ptr + n + 1, 0);
    for (i64 p = 0; p < nnz; p++) row_ptr[row_idx[p] + 1]++;
    for (i64 i = 0; i < n; i++) row_ptr[i + 1] += row_ptr[i];
    std::vector<i64> fill(row_ptr, row_ptr + n);
    // columns visited in ascending order => ascending columns within each row
    // (the stable argsort of sparse.py:275-277)
    for (i64 j = 0; j < n; j++) {
        for (i64 p = col_ptr[j]; p < col_ptr[j + 1]; p++) {
            i64 t = fill[row_idx[p]]++;
            col_idx[t] = j;
            csc_pos[t] = p;
        }
    }
}

extern "C" int64_t glu_csr_view(int64_t n, const int64_t *col_ptr, const int64_t *row_idx,
                                int64_t *row_ptr, int64_t *col_idx, int64_t *csc_pos) {
    if (n < 0) { set_error("n < 0"); return GLU_EINVAL; }
    build_csr(n, col_ptr, row_idx, row_ptr, col_idx, csc_pos);
    return GLU_OK;
}

extern "C" int64_t glu_symbolic_fillin(int64_t n, const int64_t *a_col_ptr,
                                       const int64_t *a_row_idx, int32_t inject_diagonal,
                                       glu_pattern **out, int64_t *injected, int64_t *bad_col,
                                       int32_t *bad_kind) {
    *out = nullptr;
    *injected = 0;
    *bad_col = -1;
    *bad_kind = 0;
    if (n < 0) { set_error("n < 0"); return GLU_EINVAL; }
    auto *pat = new glu_pattern();
    pat->n = n;
    pat->col_ptr.assign(n + 1, 0);
    pat->diag_pos.assign(n, 0);
    std::vector<i64> &rows = pat->row_idx;
    rows.reserve((size_t)std::max<i64>(2 * a_col_ptr[n], 16));
    std::vector<i64> visited(n, -1), stack, scratch, arow;
    std::vector<i64> l_lo(n, 0), l_hi(n, 0);  // traversal range of L(:,k) (pruned)
    std::vector<char> pruned(n, 0);
    stack.reserve(n);
    scratch.reserve(n);
    for (i64 j = 0; j < n; j++) {
        i64 alo = a_col_ptr[j], ahi = a_col_ptr[j + 1];
        if (ahi == alo) {
            *bad_col = j; *bad_kind = 1;
            set_error("column " + std::to_string(j) + " is structurally empty (singular)");
            delete pat;
            return GLU_ESTRUCT;
        }
        arow.assign(a_row_idx + alo, a_row_idx + ahi);
        if (std::find(arow.begin(), arow.end(), j) == arow.end()) {
            if (!inject_diagonal) {
                *bad_col = j; *bad_kind = 2;
                set_error("structural diagonal missing in column " + std::to_string(j));
                delete pat;
                return GLU_ESTRUCT;
            }
            (*injected)++;
            arow.push_back(j);
        }
        scratch.clear();
        for (i64 r : arow) {
            if (visited[r] == j) continue;
            visited[r] = j;
            stack.clear();
            stack.push_back(r);
            while (!stack.empty()) {
                i64 k = stack.back();
                stack.pop_back();
                scratch.push_back(k);
                if (k < j) {
                    for (i64 q = l_lo[k]; q < l_hi[k]; q++) {
                        i64 i = rows[q];
                        if (visited[i] != j) {
                            visited[i] = j;
                            stack.push_back(i);
                        }
                    }
                }
            }
        }
        std::sort(scratch.begin(), scratch.end());
        i64 start = (i64)rows.size();
        rows.insert(rows.end(), scratch.begin(), scratch.end());
        i64 end = (i64)rows.size();
        pat->col_ptr[j + 1] = end;
        i64 d = start + (i64)(std::lower_bound(scratch.begin(), scratch.end(), j) - scratch.begin());
        pat->diag_pos[j] = d;
        l_lo[j] = d + 1;
        l_hi[j] = end;
        // symmetric pruning with s = j: for every U(k,j) != 0 (k < j) whose
        // L(:,k) contains row j, keep only L(:,k) rows <= j for traversal.
        for (i64 p = start; p < d; p++) {
            i64 k = rows[p];
            if (pruned[k]) continue;
            const i64 *b = rows.data() + l_lo[k], *e = rows.data() + l_hi[k];
            const i64 *it = std::lower_bound(b, e, j);
            if (it != e && *it == j) {
                l_hi[k] = (i64)(it - rows.data()) + 1;
                pruned[k] = 1;
            }
        }
    }
    rows.shrink_to_fit();
    i64 nnz = (i64)rows.size();
    pat->row_ptr.resize(n + 1);
    pat->col_idx.resize(nnz);
    pat->csc_pos.resize(nnz);
    build_csr(n, pat->col_ptr.data(), rows.data(), pat->row_ptr.data(), pat->col_idx.data(),
              pat->csc_pos.data());
    *out = pat;
    return GLU_OK;
}

extern "C" int64_t glu_pattern_nnz(const glu_pattern *p) { return p ? (int64_t)p->row_idx.size() : 0; }

extern "C" void glu_pattern_export(const glu_pattern *p, int64_t *col_ptr, int64_t *row_idx,
                                   int64_t *diag_pos, int64_t *row_ptr, int64_t *col_idx,
                                   int64_t *csc_pos) {
    auto cp = [](const std::vector<i64> &v, int64_t *dst) {
        if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(i64));
    };
    cp(p->col_ptr, col_ptr);
    cp(p->row_idx, row_idx);
    cp(p->diag_pos, diag_pos);
    cp(p->row_ptr, row_ptr);
    cp(p->col_idx, col_idx);
    cp(p->csc_pos, csc_pos);
}

extern "C" void glu_pattern_free(glu_pattern *p) { delete p; }

// ---------------------------------------------------------------------------
// Dependency detection (depgraph.py:96-126) and levelization
// (depgraph.py:159-170).  Column k depends on
//   upward:  every i < k with U(i,k) != 0 and a non-empty L(:,i)
//   relaxed: upward  U  every i < k with L(k,i) != 0 (row k left of diag)
// Both sources are ascending lists, so a merge yields the sorted unique
// list that np.unique produces in the reference.
// ---------------------------------------------------------------------------
extern "C" int64_t glu_detect_relaxed(int64_t n, const int64_t *col_ptr, const int64_t *row_idx,
                                      const int64_t *diag_pos, const int64_t *row_ptr,
                                      const int64_t *col_idx, int64_t *dep_ptr,
                                      int64_t *dep_idx) {
    i64 e = 0;
    dep_ptr[0] = 0;
    for (i64 k = 0; k < n; k++) {
        i64 a = col_ptr[k], ae = diag_pos[k];        // U rows of column k (ascending)
        i64 b = row_ptr[k], be = row_ptr[k + 1];      // row k columns (ascending)
        while (true) {
            // skip U rows whose L column is empty
            while (a < ae && !(col_ptr[row_idx[a] + 1] - diag_pos[row_idx[a]] > 1)) a++;
            bool ha = a < ae;
            bool hb = b < be && col_idx[b] < k;
            if (!ha && !hb) break;
            i64 x;
            if (ha && (!hb || row_idx[a] <= col_idx[b])) {
                x = row_idx[a];
                if (hb && col_idx[b] == x) b++;
                a++;
            } else {
                x = col_idx[b];
                b++;
            }
            dep_idx[e++] = x;
        }
        dep_ptr[k + 1] = e;
    }
    return e;
}

extern "C" int64_t glu_detect_upward(int64_t n, const int64_t *col_ptr, const int64_t *row_idx,
                                     const int64_t *diag_pos, int64_t *dep_ptr, int64_t *dep_idx) {
    i64 e = 0;
    dep_ptr[0] = 0;
    for (i64 k = 0; k < n; k++) {
        for (i64 p = col_ptr[k]; p < diag_pos[k]; p++) {
            i64 i = row_idx[p];
            if (col_ptr[i + 1] - diag_pos[i] > 1) dep_idx[e++] = i;
        }
        dep_ptr[k + 1] = e;
    }
    return e;
}

// depgraph.py:129-156 detect_double_u_exact (the GLU2.0 detector the
// relaxed rule replaces; a debugging oracle): column t depends on i (L(t,i)
// != 0) when some j in {t} u L(:,t) has row j sharing a column k > t with
// row i, plus the upward edges.  Per column t the columns k > t of the rows
// {t} u L(:,t) are stamped once, then each candidate row i is scanned for a
// stamped column -- the same union the reference's per-j set intersections
// test.  dep_idx needs nnz entries.  Returns the edge count.
extern "C" int64_t glu_detect_double_u_exact(int64_t n, const int64_t *col_ptr, const int64_t *row_idx,
                                             const int64_t *diag_pos, const int64_t *row_ptr,
                                             const int64_t *col_idx, int64_t *dep_ptr, int64_t *dep_idx) {
    std::vector<i64> stamp(n, -1), cand;
    i64 e = 0;
    dep_ptr[0] = 0;
    auto mark_row = [&](i64 j, i64 t) {
        for (i64 q = row_ptr[j + 1] - 1; q >= row_ptr[j] && col_idx[q] > t; q--) stamp[col_idx[q]] = t;
    };
    for (i64 t = 0; t < n; t++) {
        cand.clear();
        for (i64 p = col_ptr[t]; p < diag_pos[t]; p++) {  // upward: U(i,t), L(:,i) non-empty
            const i64 i = row_idx[p];
            if (col_ptr[i + 1] - diag_pos[i] > 1) cand.push_back(i);
        }
        mark_row(t, t);
        for (i64 p = diag_pos[t] + 1; p < col_ptr[t + 1]; p++) mark_row(row_idx[p], t);
        for (i64 q = row_ptr[t]; q < row_ptr[t + 1] && col_idx[q] < t; q++) {  // L(t,i) != 0
            const i64 i = col_idx[q];
            bool found = false;
            for (i64 r = row_ptr[i + 1] - 1; r >= row_ptr[i] && col_idx[r] > t && !found; r--)
                found = stamp[col_idx[r]] == t;
            if (found) cand.push_back(i);
        }
        std::sort(cand.begin(), cand.end());
        cand.erase(std::unique(cand.begin(), cand.end()), cand.end());
        for (i64 i : cand) dep_idx[e++] = i;
        dep_ptr[t + 1] = e;
    }
    return e;
}

extern "C" int64_t glu_levelize(int64_t n, const int64_t *dep_ptr, const int64_t *dep_idx,
                                int64_t *level_of, int64_t *level_ptr, int64_t *level_cols) {
    i64 nl = 0;
    for (i64 j = 0; j < n; j++) {
        i64 lv = 0;
        for (i64 t = dep_ptr[j]; t < dep_ptr[j + 1]; t++) lv = std::max(lv, level_of[dep_idx[t]] + 1);
        level_of[j] = lv;
        nl = std::max(nl, lv + 1);
    }
    if (n == 0) nl = 0;
    std::fill(level_ptr, level_ptr + nl + 1, 0);
    for (i64 j = 0; j < n; j++) level_ptr[level_of[j] + 1]++;
    for (i64 l = 0; l < nl; l++) level_ptr[l + 1] += level_ptr[l];
    std::vector<i64> fill(level_ptr, level_ptr + std::max<i64>(nl, 1));
    for (i64 j = 0; j < n; j++) level_cols[fill[level_of[j]]++] = j;  // ascending within level
    return nl;
}

extern "C" int64_t glu_scatter_values(int64_t n, const int64_t *a_col_ptr,
                                      const int64_t *a_row_idx, const double *a_vals,
                                      const int64_t *f_col_ptr, const int64_t *f_row_idx,
                                      double *out) {
    std::fill(out, out + f_col_ptr[n], 0.0);
    for (i64 j = 0; j < n; j++) {
        i64 q = f_col_ptr[j], hi = f_col_ptr[j + 1];
        for (i64 p = a_col_ptr[j]; p < a_col_ptr[j + 1]; p++) {
            i64 r = a_row_idx[p];
            while (q < hi && f_row_idx[q] < r) q++;
            if (q >= hi || f_row_idx[q] != r) return j;
            out[q] = a_vals[p];
            q++;
        }
    }
    return GLU_OK;
}

// ---------------------------------------------------------------------------
// Caller schedules (factor_parallel accepts any LevelSchedule,
// numeric.py:241-351).  The update plan orders MACs by phase, so a caller's
// levels are checked, and for contract B refined, before planning:
//
//  * a source column i of column j (i in U(:,j), L(:,i) non-empty) in a
//    LATER level than j: the reference then reads j before i's updates
//    reach it (left_columns pulls an unfinished source; push_updates_owned
//    pushes an unfinished column that is divided before its last update) --
//    values the dataflow kernel cannot reproduce.  GLU_ESTRUCT, bad={i,j}.
//  * contract B, same level: the reference's single owner applies a level's
//    sources in ascending order (_kernels.py:119-149), so a later source j
//    of the level sees an earlier one's MACs into its own column or into
//    its multipliers U(j,k) (i writes (j,k) when L(j,i) != 0 and k > j is in
//    U(i,:)).  Such a level is cut into sub-levels of consecutive columns
//    at every j that depends that way on a column of its current sub-level:
//    per target the MACs keep the level-major, ascending-source order, and
//    each multiplier is read after exactly the MACs that precede it.
//
// Contract A values are schedule independent (left-looking order), so its
// phases are the caller's levels unchanged (the caller plans on the relaxed
// schedule).  Writes phase_of[n]; returns the phase count or GLU_ESTRUCT.
// ---------------------------------------------------------------------------
extern "C" int64_t glu_schedule_refine(int64_t n, const int64_t *col_ptr, const int64_t *row_idx,
                                       const int64_t *diag_pos, const int64_t *row_ptr,
                                       const int64_t *col_idx, const int64_t *level_of,
                                       int32_t contract, int64_t *phase_of, int64_t *bad) {
    bad[0] = bad[1] = -1;
    auto has_l = [&](i64 c) { return col_ptr[c + 1] - diag_pos[c] > 1; };
    i64 n_levels = 0;
    for (i64 j = 0; j < n; j++) {
        if (level_of[j] < 0) {
            set_error("negative level");
            return GLU_EINVAL;
        }
        n_levels = std::max(n_levels, level_of[j] + 1);
        for (i64 m = col_ptr[j]; m < diag_pos[j]; m++) {
            const i64 i = row_idx[m];
            if (has_l(i) && level_of[i] > level_of[j]) {
                bad[0] = i;
                bad[1] = j;
                set_error("a source column sits in a later level than its target");
                return GLU_ESTRUCT;
            }
        }
    }
    if (contract != GLU_CONTRACT_B) {
        for (i64 j = 0; j < n; j++) phase_of[j] = level_of[j];
        return n_levels;
    }
    // last U column of every row (row i's U part ends at its last CSR entry)
    std::vector<i64> cnt(n_levels + 1, 0), order(n);
    for (i64 j = 0; j < n; j++) cnt[level_of[j] + 1]++;
    for (i64 l = 0; l < n_levels; l++) cnt[l + 1] += cnt[l];
    for (i64 j = 0; j < n; j++) order[cnt[level_of[j]]++] = j;  // ascending within a level
    std::vector<i64> sub(n, -1);
    i64 phase = -1;
    for (i64 l = 0, x = 0; l < n_levels; l++) {
        const i64 end = x + (l == 0 ? cnt[0] : cnt[l] - cnt[l - 1]);
        phase++;
        for (; x < end; x++) {
            const i64 j = order[x];
            bool cut = false;
            for (i64 m = col_ptr[j]; m < diag_pos[j] && !cut; m++) {
                const i64 i = row_idx[m];
                cut = sub[i] == phase && has_l(i);
            }
            if (!cut && has_l(j)) {
                for (i64 t = row_ptr[j]; t < row_ptr[j + 1] && !cut; t++) {
                    const i64 i = col_idx[t];
                    if (i >= j) break;
                    cut = sub[i] == phase && col_idx[row_ptr[i + 1] - 1] > j;
                }
            }
            if (cut) phase++;
            sub[j] = phase;
        }
    }
    for (i64 j = 0; j < n; j++) phase_of[j] = sub[j];
    return phase + 1;
}

// ---------------------------------------------------------------------------
// Schedule hazards (the condition depgraph.py:173-205 simulates): in one
// level, writer w updates (i,k) for i in L(:,w), k in subcolumns(w); a
// same-level column r reads (r,k') for k' > r and (i',r) for i' > r.  So
// (i,k) is a hazard against reader i when level(i) == level(w) and k > i,
// and against reader k when level(k) == level(w) and i > k.  Output rows
// {level, writer, reader, i, k}, sorted like the reference's report.
// ---------------------------------------------------------------------------
extern "C" int64_t glu_find_hazards(int64_t n, const int64_t *col_ptr, const int64_t *row_idx,
                                    const int64_t *diag_pos, const int64_t *row_ptr,
                                    const int64_t *col_idx, const int64_t *level_of,
                                    int64_t max_out, int64_t *out) {
    struct H { i64 l, w, r, i, k; };
    std::vector<H> hz;
    for (i64 w = 0; w < n; w++) {
        const i64 lw = level_of[w];
        for (i64 t = row_ptr[w]; t < row_ptr[w + 1]; t++) {
            const i64 k = col_idx[t];
            if (k <= w) continue;
            for (i64 p = diag_pos[w] + 1; p < col_ptr[w + 1]; p++) {
                const i64 i = row_idx[p];
                if (level_of[i] == lw && k > i) hz.push_back({lw, w, i, i, k});
                if (level_of[k] == lw && i > k) hz.push_back({lw, w, k, i, k});
                if ((i64)hz.size() > 4 * std::max<i64>(max_out, 1) + 1000000) goto sort;
            }
        }
    }
sort:
    std::sort(hz.begin(), hz.end(), [](const H &a, const H &b) {
        if (a.l != b.l) return a.l < b.l;
        if (a.w != b.w) return a.w < b.w;
        if (a.r != b.r) return a.r < b.r;
        if (a.i != b.i) return a.i < b.i;
        return a.k < b.k;
    });
    const i64 m = std::min<i64>(max_out, (i64)hz.size());
    for (i64 x = 0; x < m; x++) {
        out[5 * x + 0] = hz[x].l; out[5 * x + 1] = hz[x].w; out[5 * x + 2] = hz[x].r;
        out[5 * x + 3] = hz[x].i; out[5 * x + 4] = hz[x].k;
    }
    return (i64)hz.size();
}

// ---------------------------------------------------------------------------
// Update plan.
//
// Right-looking GLU3.0 (paper Alg. 2, _kernels.py:119-149) applies, for
// every source column j and every subcolumn k (U(j,k) != 0, k > j), the
// MACs  A_s(i,k) -= (A_s(i,j) / A_s(j,j)) * A_s(j,k)  for i in L(:,j).
// The plan fixes, for every target slot, the order of its MACs:
//
//   contract B  every MAC of source j runs in the phase of level(j); inside
//               a phase a target receives its MACs in ascending j.  This is
//               factor_parallel(deterministic=False) bit for bit.
//   contract A  a MAC (j -> (i,k)) runs in phase max{level(j') : j' <= j a
//               source of (i,k)}, so each target receives its MACs in
//               ascending j overall: left-looking order, i.e.
//               factor_left_looking / factor_right_looking_seq /
//               factor_parallel(deterministic=True) bit for bit.  Deferring
//               a MAC past level(j) is safe: every consumer of (i,k) sits in
//               a level above all of its sources (relaxed dependencies).
//
// Values are never divided in place during the phases (the division runs on
// the fly inside each MAC, exactly as push_updates_owned does), so deferred
// MACs read the same undivided L values; one final pass pivot-checks and
// divides every column.
//
// Work units, one warp each, for one destination column k in one phase:
//   kDeep  a single target that receives >= deep_min MACs in the phase (the
//          rows/columns of power/ground hubs): its ordered contributions are
//          listed explicitly, the warp forms 32 products at a time and runs
//          the subtraction chain in registers -- one load and one store of
//          the target instead of one round trip per MAC.
//   kPush  a set of <= 128 distinct targets of column k (a position range
//          cut so the item carries <= T MACs in <= 32 chunks), with its
//          ordered chunks (contiguous runs of one source's L entries).  Per
//          MAC the plan stores a u8 index into the item's sorted target list
//          (u16 offsets), so the warp loads every target once into shared
//          memory, applies the chunks there and writes every target back
//          once.  Chunks are grouped into epochs of pairwise target-disjoint
//          chunks (kEpochBit marks an epoch start); only epochs are ordered.
// One warp owns every MAC of a target in a phase, so ordering needs no
// atomics.  T adapts to the phase's total MACs (enough items to fill the
// grid's warps, 32 <= T <= 128) unless max_item_macs fixes it.
// ---------------------------------------------------------------------------
namespace {

struct RawChunk {
    i32 lvl;
    i32 m, d, p0, cnt;
};

constexpr int kMaxItemCols = 4;  // destination columns one merged push item may cover
constexpr i64 kMaxSpanSlots = 65535;  // u16 target offsets of a merged item
constexpr i64 kMergeCols = 64;        // merge window (columns) of the plan workers

struct LocalItem {
    i32 lvl;
    i32 k;      // first destination column
    i32 ncols;  // destination columns (1..kMaxItemCols)
    i32 cols[kMaxItemCols];
    i32 kind;
    i64 base;    // kPush: slot the target offsets are relative to; kDeep: target slot
    i64 macs;
    i64 c0, c1;  // kPush: chunk range (thread-local); kDeep: deep range (thread-local)
    i64 m0;      // kPush: first map entry (thread-local)
    i64 t0, t1;  // kPush: target range (thread-local)
};

struct ThreadOut {
    std::vector<LocalItem> items;
    std::vector<glu::Chunk> chunks;
    std::vector<glu::DeepRef> deep;
    std::vector<uint8_t> map8;
    std::vector<uint16_t> tgt16;
    i64 deferred = 0;
    bool mismatch = false;
    i64 mismatch_col = -1;
};

// Emits the push items of one segment (pieces in MAC order, all targets in
// column k), bisecting by target position until every item fits
// (<= T MACs, <= 32 chunks).  A single position that still does not fit
// becomes a deep item.
struct PushEmitter {
    ThreadOut &o;
    const i64 *row_idx;
    const std::vector<i32> &posmap;
    i64 cb;      // column start slot
    i32 k, lvl;
    i64 T;
    std::vector<i32> pos_scratch, stamp;

    i32 pos_of(i32 p) const { return posmap[row_idx[p]]; }

    void emit(std::vector<glu::Chunk> &pieces) {
        i64 macs = 0;
        for (auto &c : pieces) macs += c.meta;
        if (macs == 0) return;
        if (macs <= T && macs <= glu::kMaxItemMacs && (i64)pieces.size() <= glu::kMaxItemChunks) {
            make_item(pieces, macs);
            return;
        }
        pos_scratch.clear();
        for (auto &c : pieces)
            for (i32 t = 0; t < c.meta; t++) pos_scratch.push_back(pos_of(c.p0 + t));
        std::sort(pos_scratch.begin(), pos_scratch.end());
        pos_scratch.erase(std::unique(pos_scratch.begin(), pos_scratch.end()), pos_scratch.end());
        if (pos_scratch.size() == 1) {  // one target: ordered chain
            LocalItem it{};
            it.lvl = lvl; it.k = k; it.kind = glu::kDeep;
            it.ncols = 1; it.cols[0] = k;
            it.base = cb + pos_scratch[0];
            it.macs = macs;
            it.c0 = (i64)o.deep.size();
            for (auto &c : pieces)
                for (i32 t = 0; t < c.meta; t++) o.deep.push_back({c.p0 + t, c.d, c.m, 0});
            it.c1 = (i64)o.deep.size();
            o.items.push_back(it);
            return;
        }
        const i32 cut = pos_scratch[pos_scratch.size() / 2];
        std::vector<glu::Chunk> left, right;
        for (auto &c : pieces) {
            i32 t = 0;
            while (t < c.meta && pos_of(c.p0 + t) < cut) t++;
            if (t > 0) left.push_back({c.m, c.d, c.p0, t});
            if (t < c.meta) right.push_back({c.m, c.d, c.p0 + t, c.meta - t});
        }
        emit(left);
        emit(right);
    }

    // A finished segment (one column, one phase) joins the phase's pending
    // merged item when the merged item stays within the item limits; small
    // segments of neighbouring columns thus share one warp task (the wide
    // phases otherwise shatter into ~10-MAC items).
    struct Pending {
        std::vector<glu::Chunk> pieces;
        std::vector<i64> slots;  // absolute target slot of every entry, in MAC order
        i32 cols[kMaxItemCols];
        i32 ncols = 0;
        i64 macs = 0, ntgt = 0, lo = 0, hi = -1;
        bool crit_dummy = false;
    };
    std::vector<Pending> pend;      // per phase
    std::vector<i32> pend_phases;   // phases with a pending item
    std::vector<i64> slot_scratch;
    bool merge = true;

    void make_item(const std::vector<glu::Chunk> &pieces, i64 macs) {
        slot_scratch.clear();
        for (auto &c : pieces)
            for (i32 t = 0; t < c.meta; t++) slot_scratch.push_back(cb + pos_of(c.p0 + t));
        std::vector<i64> uniq(slot_scratch);
        std::sort(uniq.begin(), uniq.end());
        uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
        const i64 ntgt = (i64)uniq.size(), lo = uniq.front(), hi = uniq.back();
        if ((i64)pend.size() <= lvl) pend.resize(lvl + 1);
        Pending &P = pend[lvl];
        if (P.macs > 0) {
            const bool same_col = P.cols[P.ncols - 1] == k;
            const bool fits = merge && P.macs + macs <= T && P.ntgt + ntgt <= glu::kMaxItemMacs &&
                              (i64)(P.pieces.size() + pieces.size()) <= glu::kMaxItemChunks &&
                              (same_col || P.ncols < kMaxItemCols) &&
                              std::max(P.hi, hi) - std::min(P.lo, lo) <= kMaxSpanSlots;
            if (!fits) flush_phase(lvl);
        }
        if (P.macs == 0) {
            P.pieces.clear();
            P.slots.clear();
            P.ncols = 0;
            P.ntgt = 0;
            P.lo = lo;
            P.hi = hi;
            pend_phases.push_back(lvl);
        }
        if (P.ncols == 0 || P.cols[P.ncols - 1] != k) P.cols[P.ncols++] = k;
        P.pieces.insert(P.pieces.end(), pieces.begin(), pieces.end());
        P.slots.insert(P.slots.end(), slot_scratch.begin(), slot_scratch.end());
        P.macs += macs;
        P.ntgt += ntgt;
        P.lo = std::min(P.lo, lo);
        P.hi = std::max(P.hi, hi);
    }

    void flush_phase(i32 l) {
        Pending &P = pend[l];
        if (P.macs == 0) return;
        std::vector<i64> uniq(P.slots);
        std::sort(uniq.begin(), uniq.end());
        uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
        const i64 lo = uniq.front();
        LocalItem it{};
        it.lvl = l;
        it.k = P.cols[0];
        it.ncols = P.ncols;
        for (int x = 0; x < P.ncols; x++) it.cols[x] = P.cols[x];
        it.kind = glu::kPush;
        it.base = lo;
        it.macs = P.macs;
        it.t0 = (i64)o.tgt16.size();
        for (i64 q : uniq) o.tgt16.push_back((uint16_t)(q - lo));
        it.t1 = (i64)o.tgt16.size();
        it.m0 = (i64)o.map8.size();
        it.c0 = (i64)o.chunks.size();
        stamp.assign(uniq.size(), -1);
        i32 ep = 0;
        bool first = true;
        size_t e = 0;
        for (auto c : P.pieces) {
            bool clash = false;
            const size_t mstart = o.map8.size();
            for (i32 t = 0; t < c.meta; t++, e++) {
                const i32 u = (i32)(std::lower_bound(uniq.begin(), uniq.end(), P.slots[e]) - uniq.begin());
                o.map8.push_back((uint8_t)u);
                clash = clash || stamp[u] == ep;
            }
            if (clash) ep++;
            for (size_t x = mstart; x < o.map8.size(); x++) stamp[o.map8[x]] = ep;
            if (clash || first) c.meta |= glu::kEpochBit;
            first = false;
            o.chunks.push_back(c);
        }
        it.c1 = (i64)o.chunks.size();
        o.items.push_back(it);
        P.macs = 0;
    }

    void flush_all() {
        for (i32 l : pend_phases) flush_phase(l);
        pend_phases.clear();
    }
};

}  // namespace

struct glu_plan {
    i64 n_levels = 0;
    std::vector<i64> level_item_ptr;
    std::vector<glu::Item> items;
    std::vector<glu::Chunk> chunks;
    std::vector<glu::DeepRef> deep;
    std::vector<uint8_t> map8;
    std::vector<uint16_t> tgt16;
    std::vector<i32> col_total;
    std::vector<glu::ColDep> cdeps;  // per item: destination columns and their earlier-phase counts
    i64 tail_t0 = 0, tail_macs = 0;
    i64 max_item_macs = 0;
    i64 max_push_macs = 0;
    i64 max_chunks = 0;
    i64 deferred = 0;
    i64 n_deep_items = 0;
    i64 n_epochs = 0;
    std::unique_ptr<glu::SnPlan> sn;  // supernodal engine (glu_plan_build_sn): no items above
};

static constexpr i64 kMaxSpan = 65535;
static constexpr i64 kTargetItemsPerPhase = 148 * 16 / 4;  // a quarter of the resident warps
static constexpr i64 kMinItemMacs = 32;

// Dense tail: the longest suffix of columns t0..n-1 that are each alone in
// their phase, in index order, and are the last phases of the schedule (at
// most tail_max columns, at least kTailMin).  Its MACs are left to the
// cluster tail kernel (glu_device.cu), which applies them column by column
// -- ascending source order, i.e. both contracts' order -- after every MAC
// of the plan (all from earlier phases and lower sources) is done.
static constexpr i64 kTailMin = 16;

static i64 find_tail(i64 n, const int64_t *level_of, i64 n_levels, i64 tail_max) {
    if (tail_max <= 0 || n == 0) return n;
    std::vector<i64> size(n_levels, 0);
    for (i64 j = 0; j < n; j++) size[level_of[j]]++;
    i64 j = n - 1;
    while (j >= 0 && n - j <= tail_max && size[level_of[j]] == 1 && level_of[j] == n_levels - (n - j)) j--;
    const i64 t0 = j + 1;
    return n - t0 >= kTailMin ? t0 : n;
}

extern "C" int64_t glu_plan_build(int64_t n, const int64_t *col_ptr, const int64_t *row_idx,
                                  const int64_t *diag_pos, const int64_t *level_of,
                                  int32_t contract, int64_t max_item_macs, int64_t deep_min,
                                  int64_t tail_max, int32_t n_threads, glu_plan **out) {
    *out = nullptr;
    if (contract != GLU_CONTRACT_A && contract != GLU_CONTRACT_B) {
        set_error("contract must be GLU_CONTRACT_A or GLU_CONTRACT_B");
        return GLU_EINVAL;
    }
    if (col_ptr[n] >= (int64_t)INT32_MAX) {
        set_error("pattern has >= 2^31 entries; slot indices are int32 on the device");
        return GLU_EINVAL;
    }
    const i64 D = deep_min > 0 ? deep_min : 32;  // measured on cfg2: 8 -> 6.69 ms, 32 -> 6.58 ms
    i64 n_levels = 0;
    for (i64 j = 0; j < n; j++) n_levels = std::max(n_levels, level_of[j] + 1);
    const i64 t0 = find_tail(n, level_of, n_levels, tail_max);
    // per-phase MAC totals (at the source's level) -> per-phase item size T
    std::vector<i64> phase_macs(n_levels, 0);
    i64 tail_macs = 0;
    for (i64 k = 0; k < n; k++)
        for (i64 m = col_ptr[k]; m < diag_pos[k]; m++) {
            const i64 j = row_idx[m];
            if (j >= t0) tail_macs += col_ptr[j + 1] - diag_pos[j] - 1;
            else phase_macs[level_of[j]] += col_ptr[j + 1] - diag_pos[j] - 1;
        }
    // Item size: every item costs one dependency wait and one round of
    // loads whatever its size (all of a lane's entries load together), so
    // items are as large as the warp allows -- except in a phase too small to
    // give every warp one, where smaller items spread the work.
    std::vector<i64> Tp(n_levels);
    for (i64 l = 0; l < n_levels; l++)
        Tp[l] = max_item_macs > 0
                    ? std::min<i64>(max_item_macs, glu::kMaxItemMacs)
                    : std::min<i64>(glu::kMaxItemMacs,
                                    std::max<i64>(kMinItemMacs, (phase_macs[l] + kTargetItemsPerPhase - 1) /
                                                                    kTargetItemsPerPhase));
    int nt = n_threads > 0 ? n_threads : (int)std::max(1u, std::thread::hardware_concurrency());
    nt = (int)std::min<i64>(nt, std::max<i64>(1, n / 64));
    std::vector<ThreadOut> outs(nt);
    std::atomic<i64> next{0};
    const i64 block = 256;

    auto worker = [&](int tid) {
        ThreadOut &o = outs[tid];
        std::vector<i32> posmap(n, -1);
        std::vector<i32> runmax;   // contract A: running max level per position
        std::vector<i64> hist;     // MACs per position in the current phase
        std::vector<i64> deepidx;  // position -> deep item (local index) or -1
        std::vector<i64> seg_of;   // position -> segment index or -1
        std::vector<RawChunk> raw;
        std::vector<std::vector<glu::Chunk>> seg_chunks;
        std::vector<std::vector<glu::DeepRef>> deep_lists;
        std::vector<i64> deep_pos;
        PushEmitter em{o, row_idx, posmap, 0, 0, 0, 0, {}, {}, {}, {}, {}, true};
        if (const char *e = std::getenv("GLU_MERGE")) em.merge = std::atoi(e) != 0;
        while (true) {
            i64 k0 = next.fetch_add(block);
            if (k0 >= n) break;
            i64 k1 = std::min<i64>(n, k0 + block);
            for (i64 k = k0; k < k1; k++) {
                if (k > k0 && (k - k0) % kMergeCols == 0) em.flush_all();
                i64 cb = col_ptr[k], ce = col_ptr[k + 1], len = ce - cb;
                raw.clear();
                bool any = false;
                for (i64 m = cb; m < diag_pos[k]; m++) {
                    i64 j = row_idx[m];
                    if (col_ptr[j + 1] - diag_pos[j] > 1) { any = true; break; }
                }
                if (!any) continue;
                for (i64 t = 0; t < len; t++) posmap[row_idx[cb + t]] = (i32)t;
                if (contract == GLU_CONTRACT_A) runmax.assign(len, -1);
                bool bad = false;
                for (i64 m = cb; m < diag_pos[k] && !bad; m++) {
                    i64 j = row_idx[m];
                    if (j >= t0) break;  // tail sources: the cluster tail kernel
                    i64 lo = diag_pos[j] + 1, hi = col_ptr[j + 1];
                    if (lo >= hi) continue;
                    i32 lj = (i32)level_of[j];
                    if (contract == GLU_CONTRACT_B) {
                        for (i64 p = lo; p < hi; p++)
                            if (posmap[row_idx[p]] < 0) { bad = true; break; }
                        raw.push_back({lj, (i32)m, (i32)diag_pos[j], (i32)lo, (i32)(hi - lo)});
                    } else {
                        i64 run0 = lo;
                        i32 run_l = -1;
                        for (i64 p = lo; p < hi; p++) {
                            i32 pos = posmap[row_idx[p]];
                            if (pos < 0) { bad = true; break; }
                            i32 l = std::max(runmax[pos], lj);
                            runmax[pos] = l;
                            if (l != lj) o.deferred++;
                            if (p == lo) run_l = l;
                            else if (l != run_l) {
                                raw.push_back({run_l, (i32)m, (i32)diag_pos[j], (i32)run0, (i32)(p - run0)});
                                run0 = p;
                                run_l = l;
                            }
                        }
                        if (!bad)
                            raw.push_back({run_l, (i32)m, (i32)diag_pos[j], (i32)run0, (i32)(hi - run0)});
                    }
                }
                if (bad) {
                    for (i64 t = 0; t < len; t++) posmap[row_idx[cb + t]] = -1;
                    if (!o.mismatch || k < o.mismatch_col) { o.mismatch = true; o.mismatch_col = k; }
                    continue;
                }
                // group by phase; stable keeps ascending source order inside a phase
                std::stable_sort(raw.begin(), raw.end(),
                                 [](const RawChunk &a, const RawChunk &b) { return a.lvl < b.lvl; });
                if ((i64)hist.size() < len) {
                    hist.assign(len, 0);
                    deepidx.assign(len, -1);
                    seg_of.assign(len, -1);
                }
                em.cb = cb;
                em.k = (i32)k;
                size_t g0 = 0;
                while (g0 < raw.size()) {
                    size_t g1 = g0;
                    while (g1 < raw.size() && raw[g1].lvl == raw[g0].lvl) g1++;
                    const i32 lvl = raw[g0].lvl;
                    const i64 T = Tp[lvl];
                    em.lvl = lvl;
                    em.T = T;
                    // MAC histogram over destination positions
                    i64 pmin = len, pmax = -1;
                    for (size_t c = g0; c < g1; c++) {
                        const RawChunk &ch = raw[c];
                        for (i32 t = 0; t < ch.cnt; t++) {
                            i32 pos = posmap[row_idx[ch.p0 + t]];
                            hist[pos]++;
                            pmin = std::min<i64>(pmin, pos);
                            pmax = std::max<i64>(pmax, pos);
                        }
                    }
                    // deep targets: positions with >= D MACs in this phase
                    deep_pos.clear();
                    for (i64 pos = pmin; pos <= pmax; pos++)
                        if (hist[pos] >= D) {
                            deepidx[pos] = (i64)deep_pos.size();
                            deep_pos.push_back(pos);
                        }
                    if ((i64)deep_lists.size() < (i64)deep_pos.size()) deep_lists.resize(deep_pos.size());
                    for (size_t x = 0; x < deep_pos.size(); x++) deep_lists[x].clear();
                    // greedy segmentation of the remaining positions by MACs and span
                    std::vector<i64> cuts;  // segment starts
                    cuts.push_back(pmin);
                    i64 acc = 0;
                    for (i64 pos = pmin; pos <= pmax; pos++) {
                        i64 h = deepidx[pos] >= 0 ? 0 : hist[pos];
                        if (h == 0) continue;
                        if ((acc > 0 && acc + h > T) || pos - cuts.back() >= kMaxSpan) {
                            cuts.push_back(pos);
                            acc = 0;
                        }
                        acc += h;
                    }
                    cuts.push_back(pmax + 1);
                    size_t nseg = cuts.size() - 1;
                    {
                        size_t s = 0;
                        for (i64 pos = pmin; pos <= pmax; pos++) {
                            while (pos >= cuts[s + 1]) s++;
                            seg_of[pos] = (i64)s;
                        }
                    }
                    if (seg_chunks.size() < nseg) seg_chunks.resize(nseg);
                    for (size_t s = 0; s < nseg; s++) seg_chunks[s].clear();
                    // split chunks at segment boundaries and around deep targets
                    for (size_t c = g0; c < g1; c++) {
                        const RawChunk &ch = raw[c];
                        i32 t = 0;
                        while (t < ch.cnt) {
                            i32 pos = posmap[row_idx[ch.p0 + t]];
                            if (deepidx[pos] >= 0) {
                                deep_lists[deepidx[pos]].push_back({ch.p0 + t, ch.d, ch.m, 0});
                                t++;
                                continue;
                            }
                            const i64 s = seg_of[pos];
                            i32 t1 = t + 1;
                            while (t1 < ch.cnt) {
                                i32 p2 = posmap[row_idx[ch.p0 + t1]];
                                if (deepidx[p2] >= 0 || seg_of[p2] != s) break;
                                t1++;
                            }
                            seg_chunks[s].push_back({ch.m, ch.d, ch.p0 + t, t1 - t});
                            t = t1;
                        }
                    }
                    for (size_t x = 0; x < deep_pos.size(); x++) {
                        LocalItem it{};
                        it.lvl = lvl;
                        it.k = (i32)k;
                        it.ncols = 1;
                        it.cols[0] = (i32)k;
                        it.kind = glu::kDeep;
                        it.base = cb + deep_pos[x];
                        it.macs = (i64)deep_lists[x].size();
                        it.c0 = (i64)o.deep.size();
                        o.deep.insert(o.deep.end(), deep_lists[x].begin(), deep_lists[x].end());
                        it.c1 = (i64)o.deep.size();
                        o.items.push_back(it);
                    }
                    for (size_t s = 0; s < nseg; s++)
                        if (!seg_chunks[s].empty()) em.emit(seg_chunks[s]);
                    for (i64 pos = pmin; pos <= pmax; pos++) {
                        hist[pos] = 0;
                        deepidx[pos] = -1;
                        seg_of[pos] = -1;
                    }
                    g0 = g1;
                }
                for (i64 t = 0; t < len; t++) posmap[row_idx[cb + t]] = -1;
            }
            em.flush_all();
        }
    };
    std::vector<std::thread> th;
    for (int t = 1; t < nt; t++) th.emplace_back(worker, t);
    worker(0);
    for (auto &t : th) t.join();

    i64 mism = -1;
    for (auto &o : outs)
        if (o.mismatch && (mism < 0 || o.mismatch_col < mism)) mism = o.mismatch_col;
    if (mism >= 0) {
        set_error("update targets a slot absent from the filled pattern (column " +
                  std::to_string(mism) + ")");
        return GLU_MISMATCH;
    }

    // Global, thread-independent order: phase, then estimated cost
    // descending (the longest items go first in the static warp round-robin;
    // a deep item's serial chain costs ~8x a push item's MAC), then column,
    // then base.
    struct Ref { i32 lvl; i32 crit; i32 tid; i64 idx; i64 cost; i32 need[kMaxItemCols]; };
    std::vector<Ref> refs;
    size_t total_items = 0, total_map = 0, total_tgt = 0, total_chunks = 0, total_deep = 0;
    for (auto &o : outs) {
        total_items += o.items.size();
        total_map += o.map8.size();
        total_tgt += o.tgt16.size();
        total_chunks += o.chunks.size();
        total_deep += o.deep.size();
    }
    if (total_chunks >= (size_t)INT32_MAX) {
        set_error("plan has >= 2^31 chunks");
        return GLU_EINVAL;
    }
    refs.reserve(total_items);
    // In phases with more items than crit_wide (~2.5 per resident warp),
    // releases are batched per warp (no immediate fence): the next phase
    // waits on many items anyway.  Measured: cfg2 6.760 -> 6.745 ms, cfg3
    // 5.011 -> 4.987 ms (GLU_CRIT_WIDE overrides, tuning)
    i64 crit_wide = 6000;
    if (const char *e = std::getenv("GLU_CRIT_WIDE")) crit_wide = std::atoll(e);
    std::vector<i64> phase_items(n_levels, 0);
    for (auto &o : outs)
        for (auto &x : o.items) phase_items[x.lvl]++;
    for (int t = 0; t < nt; t++)
        for (i64 i = 0; i < (i64)outs[t].items.size(); i++) {
            const LocalItem &x = outs[t].items[i];
            // critical: a destination is a source column of the next phase
            i32 crit = 0;
            for (int c = 0; c < x.ncols; c++) crit |= level_of[x.cols[c]] == x.lvl + 1 ? 1 : 0;
            if (phase_items[x.lvl] > crit_wide) crit = 0;
            refs.push_back({x.lvl, crit, t, i, x.kind == glu::kDeep ? 8 * x.macs : x.macs, {0, 0, 0, 0}});
        }
    // inside a phase: deep chains first (the longest serial work), then the
    // items the next phase waits for, then by cost
    std::sort(refs.begin(), refs.end(), [&](const Ref &a, const Ref &b) {
        if (a.lvl != b.lvl) return a.lvl < b.lvl;
        const bool da = outs[a.tid].items[a.idx].kind == glu::kDeep;
        const bool db = outs[b.tid].items[b.idx].kind == glu::kDeep;
        if (da != db) return da;
        if (a.crit != b.crit) return a.crit > b.crit;
        if (a.cost != b.cost) return a.cost > b.cost;
        const LocalItem &x = outs[a.tid].items[a.idx], &y = outs[b.tid].items[b.idx];
        if (x.k != y.k) return x.k < y.k;
        return x.base < y.base;
    });
    // dataflow dependencies (on the phase-sorted order): per item, the items
    // into its column in earlier phases; per column, the items into it overall
    std::vector<i32> cnt_k(n, 0), pend_k(n, 0), last_k(n, -1);
    for (auto &r : refs) {
        const LocalItem &x = outs[r.tid].items[r.idx];
        for (int c = 0; c < x.ncols; c++) {
            const i32 k = x.cols[c];
            if (last_k[k] != x.lvl) {
                cnt_k[k] += pend_k[k];
                pend_k[k] = 0;
                last_k[k] = x.lvl;
            }
            r.need[c] = cnt_k[k];
            pend_k[k]++;
        }
    }
    auto *plan = new glu_plan();
    plan->n_levels = n_levels;
    plan->tail_t0 = t0;
    plan->tail_macs = tail_macs;
    plan->level_item_ptr.assign(n_levels + 1, 0);
    plan->items.reserve(refs.size());
    plan->chunks.reserve(total_chunks);
    plan->map8.reserve(total_map);
    plan->tgt16.reserve(total_tgt);
    plan->deep.reserve(total_deep);
    for (auto &r : refs) {
        const ThreadOut &o = outs[r.tid];
        const LocalItem &x = o.items[r.idx];
        plan->level_item_ptr[x.lvl + 1]++;
        glu::Item it{};
        it.col = (i32)plan->cdeps.size();  // its (column, need) list
        it.need = x.ncols;
        for (int c = 0; c < x.ncols; c++) plan->cdeps.push_back({x.cols[c], r.need[c]});
        it.base = (i32)x.base;
        it.macs = (i32)x.macs;
        // phase in the upper bits (dataflow waits); bit 1: critical (signal at once)
        it.kind = (x.lvl << 2) | (r.crit << 1) | x.kind;
        if (x.kind == glu::kDeep) {
            it.map_off = (i64)plan->deep.size();
            plan->deep.insert(plan->deep.end(), o.deep.begin() + x.c0, o.deep.begin() + x.c1);
            plan->n_deep_items++;
        } else {
            it.map_off = (i64)plan->map8.size();
            plan->map8.insert(plan->map8.end(), o.map8.begin() + x.m0, o.map8.begin() + x.m0 + x.macs);
            it.tgt_off = (i64)plan->tgt16.size();
            plan->tgt16.insert(plan->tgt16.end(), o.tgt16.begin() + x.t0, o.tgt16.begin() + x.t1);
            it.ntgt = (i32)(x.t1 - x.t0);
            it.c0 = (i32)plan->chunks.size();
            for (i64 c = x.c0; c < x.c1; c++) {
                glu::Chunk ch = o.chunks[c];
                if (ch.meta & glu::kEpochBit) plan->n_epochs++;
                // pivot slot -> source column (the device waits on it)
                ch.d = (i32)(std::upper_bound(col_ptr, col_ptr + n + 1, (i64)ch.d) - col_ptr - 1);
                plan->chunks.push_back(ch);
            }
            it.nch = (i32)(x.c1 - x.c0);
            plan->max_chunks = std::max<i64>(plan->max_chunks, x.c1 - x.c0);
            plan->max_push_macs = std::max<i64>(plan->max_push_macs, x.macs);
        }
        plan->max_item_macs = std::max<i64>(plan->max_item_macs, x.macs);
        plan->items.push_back(it);
    }
    for (i64 l = 0; l < n_levels; l++) plan->level_item_ptr[l + 1] += plan->level_item_ptr[l];
    plan->col_total.resize(n);
    for (i64 k = 0; k < n; k++) plan->col_total[k] = cnt_k[k] + pend_k[k];
    for (auto &o : outs) plan->deferred += o.deferred;
    *out = plan;
    return GLU_OK;
}

extern "C" void glu_plan_info(const glu_plan *p, int64_t *info) {
    info[0] = p->n_levels;
    info[1] = (i64)p->items.size();
    info[2] = (i64)p->chunks.size();
    info[3] = (i64)p->map8.size() + (i64)p->deep.size() + p->tail_macs;
    info[4] = p->max_item_macs;
    info[5] = p->max_chunks;
    info[6] = p->deferred;
    info[7] = (i64)(p->items.size() * sizeof(glu::Item) + p->chunks.size() * sizeof(glu::Chunk) +
                    p->level_item_ptr.size() * sizeof(i64) + p->map8.size() +
                    p->tgt16.size() * sizeof(uint16_t) + p->deep.size() * sizeof(glu::DeepRef));
    info[8] = p->n_deep_items;
    info[9] = (i64)p->deep.size();
    info[10] = p->n_epochs;
    info[11] = (i64)p->map8.size();
    info[12] = (i64)p->tgt16.size();
    info[13] = p->tail_t0;
    info[14] = p->tail_macs;
    info[15] = 0;  // reserved (was the express-queue item count)
}

extern "C" void glu_plan_export(const glu_plan *p, int64_t *level_item_ptr, int64_t *items,
                                int64_t *chunks, int64_t *deep, uint8_t *map8, int64_t *tgt) {
    if (level_item_ptr)
        std::memcpy(level_item_ptr, p->level_item_ptr.data(), p->level_item_ptr.size() * sizeof(i64));
    // items in phase order (the device array's order); level_item_ptr
    // indexes this order
    std::vector<i64> order(p->items.size());
    for (size_t i = 0; i < order.size(); i++) order[i] = (i64)i;
    std::stable_sort(order.begin(), order.end(), [&](i64 x, i64 y) {
        return (p->items[x].kind >> 2) < (p->items[y].kind >> 2);
    });
    if (items)
        for (size_t i = 0; i < p->items.size(); i++) {
            const glu::Item &it = p->items[order[i]];
            i64 *o = items + 8 * i;
            o[0] = it.map_off; o[1] = it.tgt_off; o[2] = it.base; o[3] = it.c0; o[4] = it.nch;
            o[5] = it.ntgt; o[6] = it.macs; o[7] = it.kind & 1;
        }
    if (chunks)
        for (size_t i = 0; i < p->chunks.size(); i++) {
            const glu::Chunk &c = p->chunks[i];
            i64 *o = chunks + 5 * i;
            o[0] = c.m; o[1] = c.d; o[2] = c.p0; o[3] = c.meta & ~glu::kEpochBit;
            o[4] = (c.meta & glu::kEpochBit) ? 1 : 0;
        }
    if (deep)
        for (size_t i = 0; i < p->deep.size(); i++) {
            const glu::DeepRef &r = p->deep[i];
            i64 *o = deep + 3 * i;
            o[0] = r.l; o[1] = r.d; o[2] = r.m;
        }
    if (map8 && !p->map8.empty()) std::memcpy(map8, p->map8.data(), p->map8.size());
    if (tgt)
        for (size_t i = 0; i < p->tgt16.size(); i++) tgt[i] = p->tgt16[i];
}

extern "C" void glu_plan_free(glu_plan *p) { delete p; }

// Supernodal plan (glu_snode.cpp): the same MACs, in the same per-target
// order (contract A), indexed per (supernode, target column) instead of per
// MAC.  The round-1 item arrays stay empty; level_of only sizes the
// per-level bookkeeping the handle keeps.
extern "C" int64_t glu_plan_build_sn(int64_t n, const int64_t *col_ptr, const int64_t *row_idx,
                                     const int64_t *diag_pos, const int64_t *row_ptr,
                                     const int64_t *col_idx, const int64_t *csc_pos,
                                     const int64_t *level_of, int32_t n_threads, glu_plan **out) {
    *out = nullptr;
    auto *plan = new glu_plan();
    plan->sn = std::make_unique<glu::SnPlan>();
    const i64 rc = glu::sn_build(n, col_ptr, row_idx, diag_pos, row_ptr, col_idx, csc_pos, n_threads,
                                 plan->sn.get());
    if (rc != GLU_OK) {
        delete plan;
        return rc;
    }
    i64 n_levels = 0;
    for (i64 j = 0; j < n; j++) n_levels = std::max<i64>(n_levels, level_of[j] + 1);
    plan->n_levels = n_levels;
    plan->level_item_ptr.assign(n_levels + 1, 0);
    plan->col_total.assign(n, 0);
    plan->tail_t0 = n;
    *out = plan;
    return GLU_OK;
}

extern "C" void glu_sn_plan_export(const glu_plan *p, int32_t *sn, int32_t *pan, int32_t *panm,
                                   int32_t *pairs, int32_t *relmap, int32_t *push, int32_t *push_need,
                                   int32_t *tasks, int32_t *col_a, int32_t *rg, int32_t *rg_slot,
                                   uint16_t *rg_idx, uint16_t *rg_uidx) {
    const glu::SnPlan *s = p->sn.get();
    if (!s) return;
    auto cp4 = [](const std::vector<glu::I4> &v, int32_t *dst) {
        if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(glu::I4));
    };
    auto cp1 = [](const std::vector<int32_t> &v, int32_t *dst) {
        if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(int32_t));
    };
    cp4(s->sn, sn); cp4(s->pan, pan); cp4(s->panm, panm); cp4(s->pairs, pairs); cp1(s->relmap, relmap);
    cp4(s->push, push); cp1(s->push_need, push_need); cp4(s->tasks, tasks); cp1(s->col_a, col_a);
    cp4(s->rg, rg); cp1(s->rg_slot, rg_slot);
    if (rg_idx && !s->rg_idx.empty()) std::memcpy(rg_idx, s->rg_idx.data(), s->rg_idx.size() * sizeof(uint16_t));
    if (rg_uidx && !s->rg_uidx.empty()) std::memcpy(rg_uidx, s->rg_uidx.data(), s->rg_uidx.size() * sizeof(uint16_t));
}

extern "C" void glu_sn_plan_info(const glu_plan *p, int64_t *info) {
    std::memset(info, 0, sizeof(int64_t) * 16);
    const glu::SnPlan *s = p->sn.get();
    if (!s) return;
    info[0] = (i64)s->sn.size();
    info[1] = (i64)s->pan.size();
    info[2] = (i64)s->pairs.size();
    info[3] = (i64)s->relmap.size();
    info[4] = (i64)s->push.size();
    info[5] = (i64)s->tasks.size() / 3;
    info[6] = s->n_dblk;
    info[7] = s->crit_ns;
    info[8] = s->macs;
    info[9] = (i64)((s->sn.size() + s->pan.size() + s->panm.size() + s->pairs.size() + s->push.size() +
                     s->tasks.size() + s->rg.size()) * sizeof(glu::I4) +
                    (s->relmap.size() + s->push_need.size() + s->col_a.size() + s->rg_slot.size()) *
                        sizeof(int32_t) +
                    (s->rg_idx.size() + s->rg_uidx.size()) * sizeof(uint16_t));
    info[10] = (i64)s->rg.size();
    info[11] = (i64)s->rg_slot.size();
    info[12] = (i64)s->rg_idx.size();
    info[13] = (i64)s->rg_uidx.size();
}

namespace glu {
const glu_plan_view plan_view(const glu_plan *p) {
    glu_plan_view v;
    v.n_levels = p->n_levels;
    v.level_item_ptr = p->level_item_ptr.data();
    v.items = p->items.data();
    v.n_items = (i64)p->items.size();
    v.chunks = p->chunks.data();
    v.n_chunks = (i64)p->chunks.size();
    v.n_map = (i64)p->map8.size();
    v.deep = p->deep.data();
    v.n_deep = (i64)p->deep.size();
    v.map8 = p->map8.data();
    v.tgt16 = p->tgt16.data();
    v.n_tgt = (i64)p->tgt16.size();
    v.col_total = p->col_total.data();
    v.tail_t0 = p->tail_t0;
    v.cdeps = p->cdeps.data();
    v.max_push_macs = p->max_push_macs;
    v.n_cdeps = (i64)p->cdeps.size();
    v.sn = p->sn.get();
    return v;
}
}  // namespace glu
