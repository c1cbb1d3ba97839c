/*
 * levlu_oracle.c -- CPU restatement of the reference's numeric hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the B200
 * product path (paper_1908_00204_b200/csrc).  Only tests/, the smoke() entry
 * point and bench.py's cpu_baseline / --impl reference legs may load it.
 * The product library never links or calls it.
 *
 * Every function restates one numba kernel or driver of the reference
 * package `levlu` 0.1.0 (/root/reference/pkg/src/levlu) statement for
 * statement: same loop orders, same two rounded operations per MAC
 * (multiply, then subtract -- compile with -ffp-contract=off, no FMA), same
 * return codes (-1 ok, >=0 failing pivot column, -2 structurally absent
 * target slot).  Pinned against fixtures produced by the reference itself
 * (tests/golden/make_golden.py -> tests/golden/<case>.npz, tests/test_oracle.py).
 *
 * Indices are int64 and values fp64, as in the reference containers
 * (levlu/sparse.py:61-62).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef int64_t i64;

/* levlu/_kernels.py:15-34 scatter_values */
i64 orc_scatter_values(i64 n, const i64 *a_colptr, const i64 *a_rows, const double *a_vals,
                       const i64 *f_colptr, const i64 *f_rows, double *out) {
    memset(out, 0, sizeof(double) * (size_t)f_colptr[n]);
    for (i64 j = 0; j < n; j++) {
        i64 q = f_colptr[j], hi = f_colptr[j + 1];
        for (i64 p = a_colptr[j]; p < a_colptr[j + 1]; p++) {
            i64 r = a_rows[p];
            while (q < hi && f_rows[q] < r) q++;
            if (q >= hi || f_rows[q] != r) return j;
            out[q] = a_vals[p];
            q++;
        }
    }
    return -1;
}

/* levlu/_kernels.py:37-76 left_columns */
i64 orc_left_columns(i64 ncols, const i64 *cols, const i64 *colptr, const i64 *rows,
                     const i64 *diagpos, double *v, double *x, double thresh) {
    for (i64 c = 0; c < ncols; c++) {
        i64 j = cols[c];
        i64 lo = colptr[j], hi = colptr[j + 1], d = diagpos[j];
        for (i64 p = lo; p < hi; p++) x[rows[p]] = v[p];
        for (i64 p = lo; p < d; p++) {
            i64 k = rows[p];
            if (colptr[k + 1] - diagpos[k] > 1) {
                double xk = x[k];
                for (i64 q = diagpos[k] + 1; q < colptr[k + 1]; q++) {
                    double prod = v[q] * xk;
                    x[rows[q]] = x[rows[q]] - prod;
                }
            }
        }
        double piv = x[j];
        double cmax = 0.0;
        for (i64 p = lo; p < hi; p++) {
            double av = fabs(x[rows[p]]);
            if (av > cmax) cmax = av;
        }
        if (fabs(piv) <= thresh * cmax) {
            for (i64 p = lo; p < hi; p++) x[rows[p]] = 0.0;
            return j;
        }
        for (i64 p = d + 1; p < hi; p++) x[rows[p]] = x[rows[p]] / piv;
        for (i64 p = lo; p < hi; p++) {
            i64 r = rows[p];
            v[p] = x[r];
            x[r] = 0.0;
        }
    }
    return -1;
}

/* levlu/_kernels.py:79-116 right_looking_seq */
i64 orc_right_looking_seq(i64 n, const i64 *colptr, const i64 *rows, const i64 *diagpos,
                          double *v, const i64 *rowptr, const i64 *rowcols, const i64 *rowpos,
                          double thresh) {
    for (i64 j = 0; j < n; j++) {
        i64 lo = colptr[j], hi = colptr[j + 1], d = diagpos[j];
        double piv = v[d];
        double cmax = 0.0;
        for (i64 p = lo; p < hi; p++) {
            double av = fabs(v[p]);
            if (av > cmax) cmax = av;
        }
        if (fabs(piv) <= thresh * cmax) return j;
        for (i64 p = d + 1; p < hi; p++) v[p] = v[p] / piv;
        for (i64 t = rowptr[j]; t < rowptr[j + 1]; t++) {
            i64 k = rowcols[t];
            if (k <= j) continue;
            double mult = v[rowpos[t]];
            i64 q = colptr[k], khi = colptr[k + 1];
            for (i64 p = d + 1; p < hi; p++) {
                i64 r = rows[p];
                while (q < khi && rows[q] < r) q++;
                if (q >= khi || rows[q] != r) return -2;
                double prod = v[p] * mult;
                v[q] = v[q] - prod;
            }
        }
    }
    return -1;
}

/* levlu/_kernels.py:119-149 push_updates_owned */
i64 orc_push_updates_owned(i64 ncols, const i64 *cols, i64 owner, i64 n_owners,
                           const i64 *colptr, const i64 *rows, const i64 *diagpos, double *v,
                           const i64 *rowptr, const i64 *rowcols, const i64 *rowpos) {
    for (i64 c = 0; c < ncols; c++) {
        i64 j = cols[c];
        i64 d = diagpos[j], hi = colptr[j + 1];
        double piv = v[d];
        for (i64 t = rowptr[j]; t < rowptr[j + 1]; t++) {
            i64 k = rowcols[t];
            if (k <= j || k % n_owners != owner) continue;
            double mult = v[rowpos[t]];
            i64 q = colptr[k], khi = colptr[k + 1];
            for (i64 p = d + 1; p < hi; p++) {
                i64 r = rows[p];
                while (q < khi && rows[q] < r) q++;
                if (q >= khi || rows[q] != r) return -2;
                double l = v[p] / piv;
                double prod = l * mult;
                v[q] = v[q] - prod;
            }
        }
    }
    return -1;
}

/* levlu/_kernels.py:152-173 divide_columns */
i64 orc_divide_columns(i64 ncols, const i64 *cols, const i64 *colptr, const i64 *rows,
                       const i64 *diagpos, double *v, double thresh) {
    (void)rows;
    for (i64 c = 0; c < ncols; c++) {
        i64 j = cols[c];
        i64 lo = colptr[j], hi = colptr[j + 1], d = diagpos[j];
        double piv = v[d];
        double cmax = 0.0;
        for (i64 p = lo; p < hi; p++) {
            double av = fabs(v[p]);
            if (av > cmax) cmax = av;
        }
        if (fabs(piv) <= thresh * cmax) return j;
        for (i64 p = d + 1; p < hi; p++) v[p] = v[p] / piv;
    }
    return -1;
}

/* levlu/_kernels.py:176-183 lower_solve_inplace */
void orc_lower_solve_inplace(i64 n, const i64 *colptr, const i64 *rows, const i64 *diagpos,
                             const double *v, double *y) {
    for (i64 j = 0; j < n; j++) {
        double yj = y[j];
        if (yj != 0.0) {
            for (i64 p = diagpos[j] + 1; p < colptr[j + 1]; p++) {
                double prod = v[p] * yj;
                y[rows[p]] = y[rows[p]] - prod;
            }
        }
    }
}

/* levlu/_kernels.py:186-197 upper_solve_inplace */
i64 orc_upper_solve_inplace(i64 n, const i64 *colptr, const i64 *rows, const i64 *diagpos,
                            const double *v, double *y) {
    for (i64 j = n - 1; j >= 0; j--) {
        double piv = v[diagpos[j]];
        if (piv == 0.0) return j;
        double xj = y[j] / piv;
        y[j] = xj;
        for (i64 p = colptr[j]; p < diagpos[j]; p++) {
            double prod = v[p] * xj;
            y[rows[p]] = y[rows[p]] - prod;
        }
    }
    return -1;
}

/* ------------------------------------------------------------------------
 * Symbolic fill-in: levlu/symbolic.py:66-89 (_reach_column) and
 * levlu/symbolic.py:92-145 (symbolic_fillin).  Returns the filled nnz, or
 * -(j+1) for a structurally empty column j, -(n+1+j) for a missing diagonal
 * when inject_diagonal == 0, INT64_MIN when fill_rows (capacity `cap`) is
 * too small.  *injected receives the number of injected diagonals.
 * ---------------------------------------------------------------------- */
static int cmp_i64(const void *a, const void *b) {
    i64 x = *(const i64 *)a, y = *(const i64 *)b;
    return (x > y) - (x < y);
}

i64 orc_symbolic_fillin(i64 n, const i64 *a_colptr, const i64 *a_rows, int inject_diagonal,
                        i64 cap, i64 *col_ptr, i64 *fill_rows, i64 *diag_pos, i64 *injected) {
    i64 *visited = (i64 *)malloc(sizeof(i64) * (size_t)(n > 0 ? n : 1));
    i64 *stack = (i64 *)malloc(sizeof(i64) * (size_t)(n > 0 ? n : 1));
    i64 *scratch = (i64 *)malloc(sizeof(i64) * (size_t)(n > 0 ? n : 1));
    i64 *arow = (i64 *)malloc(sizeof(i64) * (size_t)(n + 1));
    i64 *l_lo = (i64 *)calloc((size_t)(n > 0 ? n : 1), sizeof(i64));
    i64 *l_hi = (i64 *)calloc((size_t)(n > 0 ? n : 1), sizeof(i64));
    char *pruned = (char *)calloc((size_t)(n > 0 ? n : 1), 1);
    i64 ret = 0;
    for (i64 i = 0; i < n; i++) visited[i] = -1;
    col_ptr[0] = 0;
    *injected = 0;
    for (i64 j = 0; j < n; j++) {
        i64 alo = a_colptr[j], ahi = a_colptr[j + 1], na = ahi - alo;
        if (na == 0) { ret = -(j + 1); goto done; }
        int has_diag = 0;
        for (i64 p = alo; p < ahi; p++) {
            arow[p - alo] = a_rows[p];
            if (a_rows[p] == j) has_diag = 1;
        }
        if (!has_diag) {
            if (!inject_diagonal) { ret = -(n + 1 + j); goto done; }
            (*injected)++;
            arow[na++] = j;
            qsort(arow, (size_t)na, sizeof(i64), cmp_i64);
        }
        /* _reach_column */
        i64 cnt = 0;
        for (i64 p = 0; p < na; p++) {
            i64 r = arow[p];
            if (visited[r] == j) continue;
            visited[r] = j;
            stack[0] = r;
            i64 top = 1;
            while (top > 0) {
                top--;
                i64 k = stack[top];
                scratch[cnt++] = k;
                if (k < j) {
                    for (i64 q = l_lo[k]; q < l_hi[k]; q++) {
                        i64 i = fill_rows[q];
                        if (visited[i] != j) {
                            visited[i] = j;
                            stack[top++] = i;
                        }
                    }
                }
            }
        }
        qsort(scratch, (size_t)cnt, sizeof(i64), cmp_i64);
        i64 start = col_ptr[j], end = start + cnt;
        if (end > cap) { ret = INT64_MIN; goto done; }
        memcpy(fill_rows + start, scratch, sizeof(i64) * (size_t)cnt);
        col_ptr[j + 1] = end;
        i64 d = start;
        while (d < end && fill_rows[d] < j) d++;
        diag_pos[j] = d;
        l_lo[j] = d + 1;
        l_hi[j] = end;
        /* Symmetric pruning (Eisenstat-Liu): for U(k,j) != 0 with j in L(:,k),
           the rows of L(:,k) below j are contained in L(:,j), so later DFS
           passes may stop L(:,k) at row j.  The reach sets -- the output --
           are unchanged; only the traversal gets shorter (the reference's
           plain DFS takes ~2 min on cfg4). */
        for (i64 q = start; q < d; q++) {
            i64 k = fill_rows[q];
            if (pruned[k]) continue;
            i64 lo = l_lo[k], hi = l_hi[k];
            while (lo < hi) {
                i64 mid = lo + (hi - lo) / 2;
                if (fill_rows[mid] < j) lo = mid + 1; else hi = mid;
            }
            if (lo < l_hi[k] && fill_rows[lo] == j) {
                l_hi[k] = lo + 1;
                pruned[k] = 1;
            }
        }
    }
    ret = col_ptr[n];
done:
    free(visited); free(stack); free(scratch); free(arow); free(l_lo); free(l_hi); free(pruned);
    return ret;
}

/* levlu/depgraph.py:83-126 detect_relaxed: column j depends on i for every
 * U(i,j) != 0 whose L(:,i) is non-empty (upward edges) and every L(j,i) != 0
 * (the L-row edges); the union, sorted and unique (the reference's
 * np.unique of src*n+dst keys), merged per column from the two sorted lists.
 * dep_idx needs room for nnz entries.  Returns the edge count. */
i64 orc_relaxed_deps(i64 n, const i64 *colptr, const i64 *rows, const i64 *diagpos,
                     const i64 *rowptr, const i64 *rowcols, i64 *dep_ptr, i64 *dep_idx) {
    i64 e = 0;
    dep_ptr[0] = 0;
    for (i64 j = 0; j < n; j++) {
        i64 a = colptr[j], ae = diagpos[j];   /* U rows of column j, ascending */
        i64 b = rowptr[j], be = rowptr[j + 1]; /* row j's columns, ascending */
        while (b < be && rowcols[b] < j) b++;
        be = b;
        b = rowptr[j];
        i64 last = -1;
        while (a < ae || b < be) {
            i64 x;
            if (a < ae && colptr[rows[a] + 1] - diagpos[rows[a]] <= 1) { a++; continue; }
            if (b >= be || (a < ae && rows[a] <= rowcols[b])) x = rows[a++];
            else x = rowcols[b++];
            if (x != last) { dep_idx[e++] = x; last = x; }
        }
        dep_ptr[j + 1] = e;
    }
    return e;
}

/* levlu/depgraph.py:159-170 levelize: level = 1 + max level of the deps;
 * levels listed in ascending column order (stable).  Returns the level
 * count; level_ptr needs n + 1 entries. */
i64 orc_levelize(i64 n, const i64 *dep_ptr, const i64 *dep_idx, i64 *level_of, i64 *level_ptr,
                 i64 *level_cols) {
    i64 nl = 0;
    for (i64 j = 0; j < n; j++) {
        i64 lv = 0;
        for (i64 q = dep_ptr[j]; q < dep_ptr[j + 1]; q++)
            if (level_of[dep_idx[q]] + 1 > lv) lv = level_of[dep_idx[q]] + 1;
        level_of[j] = lv;
        if (lv + 1 > nl) nl = lv + 1;
    }
    for (i64 l = 0; l <= nl; l++) level_ptr[l] = 0;
    for (i64 j = 0; j < n; j++) level_ptr[level_of[j] + 1]++;
    for (i64 l = 0; l < nl; l++) level_ptr[l + 1] += level_ptr[l];
    i64 *fill = (i64 *)malloc(sizeof(i64) * (size_t)(nl > 0 ? nl : 1));
    for (i64 l = 0; l < nl; l++) fill[l] = level_ptr[l];
    for (i64 j = 0; j < n; j++) level_cols[fill[level_of[j]]++] = j;
    free(fill);
    return nl;
}

/* ------------------------------------------------------------------------
 * factor_parallel: levlu/numeric.py:241-351.  Levels run in order; within a
 * level, `caps[l]` workers (persistent threads, two barrier waits per level
 * like _WorkCrew, levlu/numeric.py:196-238) run either
 *   deterministic: left_columns(cols[w::cap])          (numeric.py:287-293)
 *   atomic:        divide_columns(prev[w::prev_cap]) then
 *                  push_updates_owned(cols, w, cap)     (numeric.py:295-315)
 * Error aggregation follows _finish (numeric.py:279-285): min over the
 * non -1 worker results; negative min -> -2.
 * ---------------------------------------------------------------------- */
typedef struct {
    i64 n;
    const i64 *colptr, *rows, *diagpos, *rowptr, *rowcols, *rowpos;
    double *v;
    double thresh;
    const i64 *level_ptr, *level_cols, *caps;
    i64 n_levels;
    int deterministic;
    int pool;
    pthread_barrier_t bar;
    /* per phase */
    const i64 *cols; i64 ncols; i64 cap;
    const i64 *prev_cols; i64 nprev; i64 prev_cap;
    int stop;
    i64 *results;
    double **work;
    i64 **slices;
} crew_t;

typedef struct { crew_t *c; int w; } crew_arg_t;

static i64 strided(const i64 *cols, i64 ncols, i64 w, i64 cap, i64 *out) {
    i64 m = 0;
    for (i64 i = w; i < ncols; i += cap) out[m++] = cols[i];
    return m;
}

static i64 run_task(crew_t *c, int w) {
    if (c->deterministic) {
        if (w >= c->cap) return -1;
        i64 m = strided(c->cols, c->ncols, w, c->cap, c->slices[w]);
        return orc_left_columns(m, c->slices[w], c->colptr, c->rows, c->diagpos, c->v,
                                c->work[w], c->thresh);
    }
    if (c->prev_cols && w < c->prev_cap) {
        i64 m = strided(c->prev_cols, c->nprev, w, c->prev_cap, c->slices[w]);
        i64 err = orc_divide_columns(m, c->slices[w], c->colptr, c->rows, c->diagpos, c->v,
                                     c->thresh);
        if (err != -1) return err;
    }
    if (w < c->cap)
        return orc_push_updates_owned(c->ncols, c->cols, w, c->cap, c->colptr, c->rows,
                                      c->diagpos, c->v, c->rowptr, c->rowcols, c->rowpos);
    return -1;
}

static void *crew_loop(void *p) {
    crew_arg_t *a = (crew_arg_t *)p;
    crew_t *c = a->c;
    for (;;) {
        pthread_barrier_wait(&c->bar);
        if (c->stop) return NULL;
        c->results[a->w] = run_task(c, a->w);
        pthread_barrier_wait(&c->bar);
    }
}

static i64 finish(const i64 *res, int pool) {
    i64 best = -1;
    int any = 0;
    for (int w = 0; w < pool; w++) {
        if (res[w] == -1) continue;
        if (!any || res[w] < best) best = res[w];
        any = 1;
    }
    if (!any) return -1;
    return best >= 0 ? best : -2;
}

static void crew_run(crew_t *c) {
    pthread_barrier_wait(&c->bar);
    /* the calling thread acts as worker 0 to save one thread switch */
    c->results[0] = run_task(c, 0);
    pthread_barrier_wait(&c->bar);
}

i64 orc_factor_parallel(i64 n, const i64 *colptr, const i64 *rows, const i64 *diagpos,
                        const i64 *rowptr, const i64 *rowcols, const i64 *rowpos, double *v,
                        i64 n_levels, const i64 *level_ptr, const i64 *level_cols,
                        const i64 *caps, int deterministic, double thresh) {
    crew_t c;
    memset(&c, 0, sizeof(c));
    c.n = n; c.colptr = colptr; c.rows = rows; c.diagpos = diagpos;
    c.rowptr = rowptr; c.rowcols = rowcols; c.rowpos = rowpos; c.v = v; c.thresh = thresh;
    c.level_ptr = level_ptr; c.level_cols = level_cols; c.caps = caps; c.n_levels = n_levels;
    c.deterministic = deterministic;
    i64 pool = 1;
    for (i64 l = 0; l < n_levels; l++) if (caps[l] > pool) pool = caps[l];
    c.pool = (int)pool;
    c.results = (i64 *)calloc((size_t)pool, sizeof(i64));
    c.work = (double **)calloc((size_t)pool, sizeof(double *));
    c.slices = (i64 **)calloc((size_t)pool, sizeof(i64 *));
    for (i64 w = 0; w < pool; w++) {
        c.work[w] = (double *)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
        c.slices[w] = (i64 *)malloc(sizeof(i64) * (size_t)(n > 0 ? n : 1));
    }
    pthread_t *th = NULL;
    crew_arg_t *args = NULL;
    if (pool > 1) {
        pthread_barrier_init(&c.bar, NULL, (unsigned)pool);
        th = (pthread_t *)calloc((size_t)pool, sizeof(pthread_t));
        args = (crew_arg_t *)calloc((size_t)pool, sizeof(crew_arg_t));
        for (int w = 1; w < pool; w++) {
            args[w].c = &c; args[w].w = w;
            pthread_create(&th[w], NULL, crew_loop, &args[w]);
        }
    }
    i64 err = -1;
    const i64 *prev = NULL; i64 nprev = 0, prev_cap = 1;
    for (i64 l = 0; l < n_levels && err == -1; l++) {
        const i64 *cols = level_cols + level_ptr[l];
        i64 ncols = level_ptr[l + 1] - level_ptr[l];
        i64 cap = caps[l];
        if (deterministic) {
            if (pool == 1 || cap <= 1) {
                err = orc_left_columns(ncols, cols, colptr, rows, diagpos, v, c.work[0], thresh);
                if (err >= 0 || err == -2) break;
                err = -1;
            } else {
                c.cols = cols; c.ncols = ncols; c.cap = cap;
                crew_run(&c);
                err = finish(c.results, c.pool);
            }
        } else {
            if (pool == 1) {
                if (prev) {
                    err = orc_divide_columns(nprev, prev, colptr, rows, diagpos, v, thresh);
                    if (err != -1) break;
                }
                err = orc_push_updates_owned(ncols, cols, 0, 1, colptr, rows, diagpos, v,
                                             rowptr, rowcols, rowpos);
            } else {
                c.cols = cols; c.ncols = ncols; c.cap = cap;
                c.prev_cols = prev; c.nprev = nprev; c.prev_cap = prev_cap;
                crew_run(&c);
                err = finish(c.results, c.pool);
            }
            prev = cols; nprev = ncols; prev_cap = cap;
        }
    }
    if (!deterministic && err == -1 && prev) {
        if (pool == 1) {
            err = orc_divide_columns(nprev, prev, colptr, rows, diagpos, v, thresh);
        } else {
            c.cols = prev; c.ncols = 0; c.cap = 0;
            c.prev_cols = prev; c.nprev = nprev; c.prev_cap = prev_cap;
            crew_run(&c);
            err = finish(c.results, c.pool);
        }
    }
    if (pool > 1) {
        c.stop = 1;
        pthread_barrier_wait(&c.bar);
        for (int w = 1; w < pool; w++) pthread_join(th[w], NULL);
        pthread_barrier_destroy(&c.bar);
        free(th); free(args);
    }
    for (i64 w = 0; w < pool; w++) { free(c.work[w]); free(c.slices[w]); }
    free(c.work); free(c.slices); free(c.results);
    return err;
}

/* levlu/numeric.py:187-193 _pattern_flops: MACs + DIVs */
i64 orc_pattern_flops(i64 n, const i64 *colptr, const i64 *rows, const i64 *diagpos, i64 *macs) {
    i64 m = 0, divs = 0;
    for (i64 j = 0; j < n; j++) {
        divs += colptr[j + 1] - diagpos[j] - 1;
        for (i64 p = colptr[j]; p < diagpos[j]; p++) {
            i64 i = rows[p];
            m += colptr[i + 1] - diagpos[i] - 1;
        }
    }
    *macs = m;
    return m + divs;
}
