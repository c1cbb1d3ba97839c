"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Each case writes tests/golden/<case>.npz holding the input matrix and
everything the reference computes for it: the filled pattern and CSR view,
relaxed and upward dependency lists, the level schedule, level stats and
modes, the factor values of every numeric path (left-looking = contract A,
factor_parallel atomic = contract B) or the failing pivot column, flop
count, and lower/upper/full solve results for a fixed right-hand side.
The fixtures pin both the C oracle (tests/test_oracle.py) and the B200
path (tests/test_gpu_parity.py) without the reference on the GPU box.
"""

from __future__ import annotations

import os
import pathlib
import sys

import numpy as np

REF = pathlib.Path("/root/reference/pkg/src")
HERE = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(REF))
sys.path.insert(1, str(HERE.parent.parent))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import levlu as lv  # noqa: E402  (the reference)

from paper_1908_00204_b200 import synthetic  # noqa: E402  (matrix generators only)


def random_dd(rng, n, density):
    """Random diagonally dominant matrix with a full diagonal (same recipe as
    the reference's tests/conftest.py random_dd_matrix)."""
    m = max(int(density * n * n), n)
    rows = np.concatenate([rng.integers(0, n, size=m), np.arange(n)])
    cols = np.concatenate([rng.integers(0, n, size=m), np.arange(n)])
    vals = np.concatenate([rng.uniform(-1.0, 1.0, size=m), np.zeros(n)])
    a = lv.to_csc(lv.Triplets(n, n, rows, cols, vals))
    rowsum = np.zeros(n)
    np.add.at(rowsum, a.row_idx, np.abs(a.values))
    v = a.values.copy()
    cols_of = np.repeat(np.arange(n), np.diff(a.col_ptr))
    d = a.row_idx == cols_of
    v[d] = rowsum[a.row_idx[d]] + 1.0
    return lv.CscMatrix(a.n, a.col_ptr, a.row_idx, v)


def banded(n, half_bw, seed):
    rng = np.random.default_rng(seed)
    rows, cols = [], []
    for o in range(-half_bw, half_bw + 1):
        idx = np.arange(max(0, -o), min(n, n - o))
        rows.append(idx + o)
        cols.append(idx)
    rows, cols = np.concatenate(rows), np.concatenate(cols)
    vals = rng.uniform(0.1, 1.0, size=len(rows))
    vals[rows == cols] += 2.0 * (2 * half_bw + 1)
    return lv.to_csc(lv.Triplets(n, n, rows, cols, vals))


def block_arrow(nblocks, bs, seed):
    rng = np.random.default_rng(seed)
    n = nblocks * bs + 1
    rows, cols, vals = [], [], []
    for b in range(nblocks):
        r, c = np.meshgrid(np.arange(bs), np.arange(bs), indexing="ij")
        rows.append((r + b * bs).ravel())
        cols.append((c + b * bs).ravel())
        vals.append(rng.uniform(0.1, 1.0, size=bs * bs))
    last = n - 1
    rows += [np.full(n - 1, last), np.arange(n - 1), [last]]
    cols += [np.arange(n - 1), np.full(n - 1, last), [last]]
    vals += [rng.uniform(0.1, 1.0, n - 1), rng.uniform(0.1, 1.0, n - 1), [1.0]]
    rows, cols, vals = map(np.concatenate, (rows, cols, vals))
    diag = rows == cols
    rowsum = np.zeros(n)
    np.add.at(rowsum, rows, np.abs(vals))
    vals[diag] += rowsum[rows[diag]]
    return lv.to_csc(lv.Triplets(n, n, rows, cols, vals))


def from_ours(m):
    return lv.CscMatrix(m.n, m.col_ptr.copy(), m.row_idx.copy(), m.values.copy())


def load_mtx(name):
    with open(f"/root/reference/pkg/tests/data/{name}") as fh:
        return lv.to_csc(lv.load_matrix_market(fh))


def graph_csr(g, n):
    lens = np.array([len(d) for d in g.deps], dtype=np.int64)
    ptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    idx = np.concatenate(g.deps).astype(np.int64) if ptr[-1] else np.empty(0, np.int64)
    return ptr, idx


def run_case(name, a, rhs_seed=0, thresh=None):
    out = {"n": a.n, "a_col_ptr": a.col_ptr, "a_row_idx": a.row_idx, "a_values": a.values}
    fp = lv.symbolic_fillin(a.pattern)
    out.update(fp_col_ptr=fp.full.col_ptr, fp_row_idx=fp.full.row_idx, fp_diag_pos=fp.diag_pos,
               csr_row_ptr=fp.csr.row_ptr, csr_col_idx=fp.csr.col_idx,
               csr_csc_pos=fp.csr.csc_pos, nz_before=fp.nz_before)
    g = lv.detect_relaxed(fp)
    out["relaxed_ptr"], out["relaxed_idx"] = graph_csr(g, a.n)
    gu = lv.detect_upward(fp)
    out["upward_ptr"], out["upward_idx"] = graph_csr(gu, a.n)
    s = lv.levelize(g)
    out["level_of"] = s.level_of
    out["level_ptr"] = np.concatenate([[0], np.cumsum([len(c) for c in s.levels])]).astype(np.int64)
    out["level_cols"] = (np.concatenate(s.levels) if s.levels else np.empty(0)).astype(np.int64)
    st = lv.level_stats(fp, s)
    out["stat_sizes"] = np.array(st.sizes, dtype=np.int64)
    out["stat_max_sub"] = np.array(st.max_subcolumns, dtype=np.int64)
    for tag, rm in (("default", lv.ResourceModel()),
                    ("b200", lv.ResourceModel(total_warps=148 * 64, memory_budget_bytes=160 << 30))):
        plans = lv.plan_schedule(s, lv.level_stats(fp, s), a.n, rm)
        out[f"modes_{tag}"] = np.array([p.mode.value for p in plans])
        out[f"wpb_{tag}"] = np.array([p.warps_per_column for p in plans], dtype=np.int64)
    plans = lv.plan_schedule(s, lv.level_stats(fp, s), a.n, lv.ResourceModel())
    kw = {} if thresh is None else {"zero_pivot_threshold": thresh}
    out["thresh"] = thresh if thresh is not None else 1e-14
    # contract A (left-looking) and contract B (atomic, 2 workers)
    try:
        lu = lv.factor_left_looking(a, fp, lv.FactorOptions(**kw))
        out["lu_a"] = lu.values
        out["fail_a"] = -1
    except lv.PivotError as e:
        out["fail_a"] = e.column
        lu = None
    try:
        out["fail_rl"] = -1
        out["lu_rl"] = lv.factor_right_looking_seq(a, fp, lv.FactorOptions(**kw)).values
    except lv.PivotError as e:
        out["fail_rl"] = e.column
    for det, tag in ((True, "det"), (False, "b")):
        try:
            lub, stats = lv.factor_parallel(a, fp, s, plans,
                                            lv.FactorOptions(deterministic=det, worker_count=2, **kw))
            out[f"lu_{tag}"] = lub.values
            out[f"fail_{tag}"] = -1
            out["flop_count"] = stats.flop_count
        except lv.PivotError as e:
            out[f"fail_{tag}"] = e.column
    if lu is not None:
        rng = np.random.default_rng(rhs_seed)
        b = rng.standard_normal(a.n)
        b[rng.uniform(size=a.n) < 0.2] = 0.0  # exercise the y[j] == 0 skip
        out["rhs"] = b
        out["y_lower"] = lv.lower_solve(lu, b)
        try:
            out["x_upper"] = lv.upper_solve(lu, out["y_lower"])
            out["x_solve"] = lv.solve(lu, b)
            out["fail_solve"] = -1
        except lv.PivotError as e:
            out["fail_solve"] = e.column
    np.savez_compressed(HERE / f"{name}.npz", **out)
    print(f"{name}: n={a.n} nnz={fp.nnz} levels={s.level_count} fail_a={out['fail_a']}")


def main():
    run_case("two_by_two", lv.to_csc(lv.Triplets(2, 2, [0, 1, 0, 1], [0, 0, 1, 1],
                                                  [4.0, 6.0, 3.0, 3.0])))
    run_case("singular_2x2", lv.to_csc(lv.Triplets(2, 2, [0, 1, 0, 1], [0, 0, 1, 1],
                                                    [1.0, 1.0, 1.0, 1.0])))
    thr = lv.to_csc(lv.Triplets(2, 2, [0, 1, 1], [0, 0, 1], [1e-8, 1.0, 1.0]))
    run_case("threshold_pass", thr)
    run_case("threshold_fail", thr, thresh=1e-6)
    run_case("conflict8", load_mtx("conflict8.mtx"))
    run_case("diag5", load_mtx("diag5.mtx"))
    for seed, n, dens in [(1, 40, 0.1), (2, 80, 0.05), (3, 120, 0.04), (5, 100, 0.05),
                          (11, 300, 0.01), (12, 500, 0.004)]:
        run_case(f"random_dd_s{seed}_n{n}", random_dd(np.random.default_rng(seed), n, dens),
                 rhs_seed=seed)
    run_case("banded_n200", banded(200, 8, 0))
    run_case("block_arrow_4x24", block_arrow(4, 24, 7))
    run_case("cfg1", from_ours(synthetic.make("cfg1")))
    # a matrix whose zero U diagonal is only found by the upper solve
    z = lv.to_csc(lv.Triplets(3, 3, [0, 1, 2, 0], [0, 1, 2, 2], [2.0, 0.0, 1.0, 1.0]))
    run_case("zero_pivot_solve", z, thresh=0.0)


if __name__ == "__main__":
    main()
