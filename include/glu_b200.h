/*
 * glu_b200.h -- C ABI of the B200-native GLU3.0 numeric-factorization path.
 *
 * Drop-in boundary for the reference package `levlu` 0.1.0.  Every entry
 * point names the reference interface it replaces (file:line relative to
 * /root/reference/pkg/src/levlu).  Plain pointers and sizes only: indices
 * are int64 (as the reference stores them, sparse.py:61-62), values fp64.
 * The caller owns every host buffer; device buffers are owned by the
 * handle, except the `*_device` calls, which operate on caller-owned device
 * memory (e.g. torch tensors) on the caller's stream.
 *
 * Status codes follow the reference kernels' return convention
 * (_kernels.py:30-34, :114, :147 and numeric.py:110-126):
 *     GLU_OK (-1)         success
 *     >= 0                failing pivot column  -> PivotError(column)
 *     GLU_MISMATCH (-2)   structurally absent slot -> PatternMismatchError
 *     GLU_ECUDA (-3)      CUDA runtime error (message: glu_last_error)
 *     GLU_EINVAL (-4)     invalid argument      (message: glu_last_error)
 *     GLU_ESTRUCT (-5)    structural error      -> SymbolicError
 * Threading: one handle per host thread / stream; distinct handles are
 * independent.  No C++ exception crosses this boundary.
 */
#ifndef GLU_B200_H
#define GLU_B200_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GLU_OK (-1)
#define GLU_MISMATCH (-2)
#define GLU_ECUDA (-3)
#define GLU_EINVAL (-4)
#define GLU_ESTRUCT (-5)

#define GLU_CONTRACT_A 0 /* ascending-source MAC order: factor_left_looking,
                            factor_right_looking_seq, factor_parallel(deterministic=True) */
#define GLU_CONTRACT_B 1 /* level-major MAC order: factor_parallel(deterministic=False) */

typedef struct glu_pattern glu_pattern; /* filled pattern (host) */
typedef struct glu_plan glu_plan;       /* per-level update plan (host) */
typedef struct glu_handle glu_handle;   /* device-resident pattern + plan */

/* Last error message of the calling thread. Returns its length. */
int64_t glu_last_error(char *buf, int64_t len);
/* Library version / build string (sm_100a). */
const char *glu_version(void);

/* ---- host analysis (computed once per pattern) ------------------------ */

/* symbolic.py:92-145 symbolic_fillin + sparse.py:267-278 make_csr_view.
   Returns GLU_OK, or GLU_ESTRUCT with *bad_col set and *bad_kind = 1 (empty
   column, symbolic.py:122) or 2 (missing diagonal, symbolic.py:124-125). */
int64_t glu_symbolic_fillin(int64_t n, const int64_t *a_col_ptr, const int64_t *a_row_idx,
                            int32_t inject_diagonal, glu_pattern **out, int64_t *injected,
                            int64_t *bad_col, int32_t *bad_kind);
int64_t glu_pattern_nnz(const glu_pattern *p);
/* Copies the pattern out: col_ptr[n+1], row_idx[nnz], diag_pos[n],
   row_ptr[n+1], col_idx[nnz], csc_pos[nnz] (CsrView, sparse.py:121-138). */
void glu_pattern_export(const glu_pattern *p, int64_t *col_ptr, int64_t *row_idx,
                        int64_t *diag_pos, int64_t *row_ptr, int64_t *col_idx,
                        int64_t *csc_pos);
void glu_pattern_free(glu_pattern *p);

/* sparse.py:267-278 make_csr_view (stable: ascending columns per row). */
int64_t glu_csr_view(int64_t n, const int64_t *col_ptr, const int64_t *row_idx,
                     int64_t *row_ptr, int64_t *col_idx, int64_t *csc_pos);

/* depgraph.py:96-126 detect_relaxed.  dep_idx must hold nnz entries (an
   upper bound).  Returns the edge count; deps of column k are
   dep_idx[dep_ptr[k]:dep_ptr[k+1]], sorted ascending, unique. */
int64_t glu_detect_relaxed(int64_t n, const int64_t *col_ptr, const int64_t *row_idx,
                           const int64_t *diag_pos, const int64_t *row_ptr,
                           const int64_t *col_idx, int64_t *dep_ptr, int64_t *dep_idx);
/* depgraph.py:96-110 detect_upward (same output convention). */
int64_t glu_detect_upward(int64_t n, const int64_t *col_ptr, const int64_t *row_idx,
                          const int64_t *diag_pos, int64_t *dep_ptr, int64_t *dep_idx);

/* depgraph.py:129-156 detect_double_u_exact (same output convention): the
   exact GLU2.0 detector, kept as a debugging oracle. */
int64_t glu_detect_double_u_exact(int64_t n, const int64_t *col_ptr, const int64_t *row_idx,
                                  const int64_t *diag_pos, const int64_t *row_ptr,
                                  const int64_t *col_idx, int64_t *dep_ptr, int64_t *dep_idx);

/* depgraph.py:159-170 levelize.  Returns the level count; level_cols lists
   the columns level by level, ascending within each level. */
int64_t glu_levelize(int64_t n, const int64_t *dep_ptr, const int64_t *dep_idx,
                     int64_t *level_of, int64_t *level_ptr, int64_t *level_cols);

/* _kernels.py:15-34 scatter_values on the host (reference semantics):
   returns GLU_OK or the first column of A with entries outside the
   filled pattern. */
int64_t glu_scatter_values(int64_t n, const int64_t *a_col_ptr, const int64_t *a_row_idx,
                           const double *a_vals, const int64_t *f_col_ptr,
                           const int64_t *f_row_idx, double *out);

/* depgraph.py:173-205 simulate_hazards, evaluated in O(MACs): same-level
   write/read conflicts of the right-looking updates under level_of.
   Writes up to max_out rows {level, writer, reader, i, k} sorted by
   (level, writer, reader, element); returns the total found. */
int64_t glu_find_hazards(int64_t n, const int64_t *col_ptr, const int64_t *row_idx,
                         const int64_t *diag_pos, const int64_t *row_ptr, const int64_t *col_idx,
                         const int64_t *level_of, int64_t max_out, int64_t *out);

/* ---- update plan: the precomputed scatter schedule -------------------- */

/* Builds the destination-owned update plan for the given level schedule
   (the precomputed replacement of the runtime merge search in
   _kernels.py:107-115 / :140-148 and of the ownership split of
   numeric.py:295-315).  contract: GLU_CONTRACT_A or GLU_CONTRACT_B.
   max_item_macs caps the MACs one push item carries (0 = adaptive per
   phase, 32..128); deep_min is the MAC count from which a target becomes
   its own register-chained item (0 = default 32).  tail_max: the trailing
   columns that are each alone in the last phases (a near-dense separator
   block) go to the thread-block-cluster tail kernel, up to tail_max of them
   (0 = no tail; glu_tail_capacity() gives the device's limit).  Returns
   GLU_OK or GLU_MISMATCH when an update targets a slot absent from the
   pattern (the condition _kernels.py:113-114 reports at run time). */
int64_t glu_plan_build(int64_t n, const int64_t *col_ptr, const int64_t *row_idx,
                       const int64_t *diag_pos, const int64_t *level_of, int32_t contract,
                       int64_t max_item_macs, int64_t deep_min, int64_t tail_max,
                       int32_t n_threads, glu_plan **out);
/* Largest dense tail (columns) the current device's cluster kernel holds in
   distributed shared memory; 0 without a CUDA device. */
int64_t glu_tail_capacity(void);
/* Page-locked host buffer of nbytes (cudaHostAlloc, portable), for LU
   values returned through glu_factor_host: the device writes them by DMA
   while the kernel runs instead of through the driver's pageable staging.
   Returns the address, or NULL (message: glu_last_error).  No counterpart
   in the reference (its factors live in host memory throughout). */
void *glu_host_alloc(int64_t nbytes);
void glu_host_free(void *p);
/* info[0..15] = n_levels, n_items, n_chunks, MACs, max_item_macs,
   max_chunks_per_item, deferred_macs (contract A), plan bytes, deep items,
   deep MACs, epochs, push MACs (= u8 map entries), target-list entries,
   tail start column t0 (n: no tail), tail MACs, 0 (reserved).  MACs (info[3]) counts
   push + deep + tail MACs. */
void glu_plan_info(const glu_plan *p, int64_t *info);
/* level_item_ptr[n_levels+1];
   items[n_items*8]   = {map_off, tgt_off, base, c0, nch, ntgt, macs, kind (0 push, 1 deep)};
   chunks[n_chunks*5] = {m (multiplier slot), j (source column), p0, cnt, epoch_start};
   deep[deep_macs*3]  = {l, d, m}  (all slots absolute);
   map8[push_macs]    = per MAC, index into its item's target list;
   tgt[targets]       = target offsets from the item's base.  Any pointer may be NULL. */
void glu_plan_export(const glu_plan *p, int64_t *level_item_ptr, int64_t *items,
                     int64_t *chunks, int64_t *deep, uint8_t *map8, int64_t *tgt);
void glu_plan_free(glu_plan *p);

/* Supernodal plan: the same MACs and per-target MAC order as a contract-A
   plan (_kernels.py:37-76 left-looking order), indexed per (fundamental
   supernode, target column) -- ~0.1 B per MAC instead of ~3 -- for patterns
   whose per-MAC plan does not fit (the G3-like cfg4: 3.8e10 MACs).  A
   handle created from it runs the supernodal kernel (panels of <= 32
   columns, dense in-panel blocks, relative row maps).  level_of is the
   caller's schedule (it orders pivot failures, numeric.py:279-285).
   Returns GLU_OK, GLU_MISMATCH (pattern not closed under fill) or
   GLU_EINVAL. */
int64_t glu_plan_build_sn(int64_t n, const int64_t *col_ptr, const int64_t *row_idx,
                          const int64_t *diag_pos, const int64_t *row_ptr, const int64_t *col_idx,
                          const int64_t *csc_pos, const int64_t *level_of, int32_t n_threads,
                          glu_plan **out);
/* info[0..13] (16 words) = supernodes, panels, (supernode, column) pairs,
   relative-map entries, pushes, tasks, diagonal-block scratch doubles,
   critical path of the plan's latency model (ns), MACs, plan bytes, RG
   tasks, RG slots, RG MAC indices, RG U indices (all 0 for a per-MAC
   plan). */
void glu_sn_plan_info(const glu_plan *p, int64_t *info);
/* Copies a supernodal plan out (sizes from glu_sn_plan_info; int32 x4
   records): sn {s0, s1, |R_S|, first pair}, pan {p0, p1, supernode, rows
   below}, panm {RECT chunks into the panel, TRSM chunks, scratch offset or
   -1, 0}, pairs {k, a, base, map}, relmap, push {panel, pair0, pair1,
   target panel}, push_need[pushes], tasks (3 records each) {code << 27 |
   chunk, source panel, p0, p1, s1, rows below the panel, pair0, pair1,
   target panel, need, 0, 0}, col_a[n], rg {first slot, slots, first MAC
   index, first U index}, rg_slot, rg_idx (u16), rg_uidx (u16).  Any
   pointer may be NULL. */
void glu_sn_plan_export(const glu_plan *p, int32_t *sn, int32_t *pan, int32_t *panm, int32_t *pairs,
                        int32_t *relmap, int32_t *push, int32_t *push_need, int32_t *tasks,
                        int32_t *col_a, int32_t *rg, int32_t *rg_slot, uint16_t *rg_idx,
                        uint16_t *rg_uidx);

/* Checks a caller's level schedule for factor_parallel (numeric.py:241-351
   accepts any LevelSchedule) and refines it for contract B.  A source
   column (U(i,j) != 0, L(:,i) non-empty) in a later level than its target
   returns GLU_ESTRUCT with bad[0] = i, bad[1] = j (the reference would read
   an unfinished column).  Contract A: phase_of = level_of.  Contract B:
   levels are cut into sub-levels of consecutive columns wherever a column
   depends on an earlier column of its own level (the reference's single
   owner applies a level's sources in ascending order, _kernels.py:119-149),
   so the phase-ordered plan reproduces the reference's reads.  Returns the
   phase count. */
int64_t glu_schedule_refine(int64_t n, const int64_t *col_ptr, const int64_t *row_idx,
                            const int64_t *diag_pos, const int64_t *row_ptr, const int64_t *col_idx,
                            const int64_t *level_of, int32_t contract, int64_t *phase_of,
                            int64_t *bad);

/* ---- device handle ---------------------------------------------------- */

/* Uploads pattern, level schedule and plan (with its u8 scatter map) to the
   current CUDA device.  Replaces the per-call
   setup of numeric.py:241-317 (caps, workspaces, crew). */
int64_t glu_create(int64_t n, const int64_t *col_ptr, const int64_t *row_idx,
                   const int64_t *diag_pos, const int64_t *row_ptr, const int64_t *col_idx,
                   const int64_t *csc_pos, const int64_t *level_of, const glu_plan *plan,
                   glu_handle **out);
void glu_destroy(glu_handle *h);
/* Options: key 1 = record per-level GPU timestamps (value 0/1; read with
   glu_level_times, FactorStats.level_times, numeric.py:321-327); key 2 =
   failing-pivot order: 0 = earliest level then min column (factor_parallel,
   numeric.py:279-285), 1 = min column (sequential paths, numeric.py:129-159). */
int64_t glu_set_option(glu_handle *h, int64_t key, int64_t value);
/* Levels that order pivot failures (key 2 = 0): the caller's schedule,
   which may differ from the one the plan was built on (contract A plans
   on the relaxed schedule). */
int64_t glu_set_fail_levels(glu_handle *h, const int64_t *level_of);
/* Diagnostics of the supernodal engine: glu_set_option(h, 15, 1) records,
   per task of the next factorization, 6 words {start, source ready, target
   ready, done (%globaltimer ns), warp, 0}; read with glu_sn_trace (returns
   the tasks written, 0 for a per-MAC handle). */
int64_t glu_sn_trace(glu_handle *h, int64_t *out, int64_t max_tasks);
/* Diagnostics: glu_set_option(h, 3, first_phase) and (h, 4, n_phases)
   record, for every item of those phases, 8 words {item | phase << 32,
   warp, t_start, t_static_loaded, t_wait_done, t_values_loaded,
   t_stored, 0} (%globaltimer ns) in the next factorization; read them
   with glu_trace_read (returns the record count). */
int64_t glu_trace_read(glu_handle *h, int64_t *out, int64_t max_records);
/* Diagnostics: glu_set_option(h, 13, 1) records %globaltimer stamps of the
   dense-tail kernel: out[0], [1], [2], [4] = CTA 0 start, columns loaded,
   panels done, columns stored and divided; then per panel p (8 + 6p ..): its owner observed
   panel p-1, applied it, finished the column sweep of p, wrote p back, published p.  Returns the word count
   copied (0 when off). */
int64_t glu_tail_trace_read(glu_handle *h, int64_t *out, int64_t max_words);
/* Diagnostics: glu_set_option(h, 8, n) records CUDA events (on the launch
   stream) around the factor kernel and the dense-tail kernel of the next n
   factorizations; after a synchronize, glu_kernel_times writes
   {factor_kernel ms, tail_kernel ms} per launch and returns the count. */
int64_t glu_kernel_times(glu_handle *h, double *ms, int64_t max_launches);
/* Per-level milliseconds of the last timed factorization; returns count. */
int64_t glu_level_times(const glu_handle *h, double *ms, int64_t len);
/* info[0..11]: n, nnz, n_levels, n_items, n_chunks, macs, device bytes,
   grid CTAs, threads/CTA, lsolve levels, usolve levels, sm count */
void glu_handle_info(const glu_handle *h, int64_t *info);

/* A -> A_s slot map for device-side scatter (_kernels.py:15-34). Returns
   GLU_OK or the first column of A with entries outside the pattern. */
int64_t glu_set_input_pattern(glu_handle *h, int64_t nz, const int64_t *a_col_ptr,
                              const int64_t *a_row_idx);

/* Device-side scatter: v[nnz] = 0; v[slot(e)] = a_vals[e].  Device ptrs. */
int64_t glu_scatter_device(glu_handle *h, const double *a_vals, double *v, void *stream);

/* Numeric factorization in place over device A_s-slot values (numeric.py:
   241-351 level loop + _kernels.py:119-173).  Returns GLU_OK, the failing
   pivot column (min column of the earliest failing level), or an error.
   Per-level GPU times are recorded when
   enabled with glu_set_option(h, 1, 1). */
int64_t glu_factor_device(glu_handle *h, double *v, double thresh, void *stream);

/* Asynchronous launch (no host synchronization, for timing loops) and the
   status read that completes it. */
int64_t glu_factor_device_async(glu_handle *h, double *v, double thresh, void *stream);
int64_t glu_factor_status(glu_handle *h, void *stream);

/* Batch refactorization (many value sets on one pattern: the Newton /
   transient steps the reference re-calls factor_parallel for).
   v (device) holds `batch` A_s-slot value sets batch-major (set b at
   v + b * nnz), factored in place in stream order; fail_cols (host, batch)
   receives GLU_OK or the failing pivot column per set.  Returns GLU_OK or
   an error code. */
int64_t glu_factor_batch_device(glu_handle *h, int64_t batch, double *v, double thresh,
                                int64_t *fail_cols, void *stream);
/* Host-buffer batch: a_vals [batch][nz] (A values in the pattern given to
   glu_set_input_pattern) in, LU values [batch][nnz] out, per-set status in
   fail_cols. */
int64_t glu_factor_batch_host(glu_handle *h, int64_t batch, const double *a_vals, double *lu_out,
                              double thresh, int64_t *fail_cols);

/* numeric.py:354-378 solve: x (device, n) holds b on entry, x on exit.
   lu (device) are factor values. Returns GLU_OK or the column of a zero
   U diagonal (_kernels.py:190-191). */
int64_t glu_solve_device(glu_handle *h, const double *lu, double *x, void *stream);
int64_t glu_lower_solve_device(glu_handle *h, const double *lu, double *x, void *stream);
int64_t glu_upper_solve_device(glu_handle *h, const double *lu, double *x, void *stream);
/* Multi-RHS solves (device): x holds nrhs right-hand sides (column r at
   x + r * ldx, ldx >= n), overwritten by the solutions; part 0 = L then U,
   1 = L only, 2 = U only.  Each column is bitwise the single-RHS result. */
int64_t glu_solve_multi_device(glu_handle *h, const double *lu, double *x, int64_t nrhs,
                               int64_t ldx, int32_t part, void *stream);
/* Batch solves: nb systems on this pattern, each with its OWN factors (set b
   at lu + b * lu_stride, e.g. the output of glu_factor_batch_device) and one
   right-hand side (x + b * ldx, overwritten with the solution); one pair of
   dataflow launches.  status[nb] (host) gets -1 per set, or the column whose
   diagonal is exactly zero (the PivotError upper_solve raises, numeric.py:
   364-373); such a set's x is unspecified.  Each solved set is bitwise
   glu_solve_device on its factors. */
int64_t glu_solve_batch_device(glu_handle *h, const double *lu, int64_t lu_stride, double *x,
                               int64_t nb, int64_t ldx, int64_t *status, void *stream);

/* End-to-end host-buffer calls (the reference-facing plugin boundary):
   H2D of A values, device scatter, factor, D2H of LU. */
int64_t glu_factor_host(glu_handle *h, const double *a_vals, double *lu_out, double thresh);
int64_t glu_solve_host(glu_handle *h, const double *lu, const double *b, double *x);

#ifdef __cplusplus
}
#endif
#endif
