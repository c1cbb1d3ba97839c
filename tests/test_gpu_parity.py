"""B200 parity: every factorization / solve entry point, through the C ABI,
against the reference's own outputs (tests/golden) and the CPU oracle."""

from __future__ import annotations

import numpy as np
import pytest

import paper_1908_00204_b200 as glu
from conftest import csc_from_golden, load_golden, pattern_from_golden
from oracle import oracle as orc

pytestmark = pytest.mark.gpu


def _analyze(a, rm=None):
    fp = glu.symbolic_fillin(a.pattern)
    s = glu.levelize(glu.detect_relaxed(fp))
    st = glu.level_stats(fp, s)
    plans = glu.plan_schedule(s, st, a.n, rm or glu.ResourceModel())
    return fp, s, plans


def test_factor_parallel_both_contracts_bitwise(golden):
    name, g = golden
    a = csc_from_golden(g)
    fp, s, plans = _analyze(a)
    thr = float(g["thresh"])
    for det, tag in ((True, "det"), (False, "b")):
        for workers in (1, 8):
            opts = glu.FactorOptions(deterministic=det, worker_count=workers,
                                     zero_pivot_threshold=thr)
            if int(g[f"fail_{tag}"]) >= 0:
                with pytest.raises(glu.PivotError) as e:
                    glu.factor_parallel(a, fp, s, plans, opts)
                assert e.value.column == int(g[f"fail_{tag}"])
            else:
                lu, stats = glu.factor_parallel(a, fp, s, plans, opts)
                assert np.array_equal(lu.values, g[f"lu_{tag}"]), (name, tag)
                assert len(stats.level_times) == s.level_count
                assert stats.level_modes == [p.mode.value for p in plans]
                assert stats.flop_count == int(g["flop_count"])


def test_sequential_entry_points_bitwise(golden):
    name, g = golden
    a = csc_from_golden(g)
    fp = glu.symbolic_fillin(a.pattern)
    opts = glu.FactorOptions(zero_pivot_threshold=float(g["thresh"]))
    for fn, tag in ((glu.factor_left_looking, "a"), (glu.factor_right_looking_seq, "rl")):
        if int(g[f"fail_{tag}"]) >= 0:
            with pytest.raises(glu.PivotError) as e:
                fn(a, fp, opts)
            assert e.value.column == int(g[f"fail_{tag}"])
        else:
            assert np.array_equal(fn(a, fp, opts).values, g[f"lu_{tag}"]), (name, tag)


def test_solves_bitwise(golden):
    name, g = golden
    if "rhs" not in g:
        pytest.skip("factorization fails for this case")
    a = csc_from_golden(g)
    fp = glu.symbolic_fillin(a.pattern)
    lu = glu.LuFactors(fp, g["lu_a"])
    y = glu.lower_solve(lu, g["rhs"])
    assert np.array_equal(y, g["y_lower"])
    assert np.array_equal(glu.upper_solve(lu, y), g["x_upper"])
    assert np.array_equal(glu.solve(lu, g["rhs"]), g["x_solve"])


def test_upper_solve_zero_diagonal():
    a = glu.to_csc(glu.Triplets(3, 3, [0, 1, 2, 0], [0, 1, 2, 2], [2.0, 3.0, 1.0, 1.0]))
    fp = glu.symbolic_fillin(a.pattern)
    vals = np.array([2.0, 0.0, 1.0, 1.0])  # U(1,1) = 0
    with pytest.raises(glu.PivotError) as e:
        glu.upper_solve(glu.LuFactors(fp, vals), np.ones(3))
    assert e.value.column == 1
    with pytest.raises(ValueError):
        glu.lower_solve(glu.LuFactors(fp, vals), np.ones(2))


def test_scatter_rejects_pattern_mismatch():
    from conftest import random_dd

    rng = np.random.default_rng(9)
    a = random_dd(rng, 15, 0.15)
    fp = glu.symbolic_fillin(a.pattern)
    bigger = random_dd(rng, 15, 0.4)
    with pytest.raises(glu.PatternMismatchError):
        glu.factor_left_looking(bigger, fp)


def test_detect_races():
    g = load_golden("conflict8")
    a = csc_from_golden(g)
    fp = glu.symbolic_fillin(a.pattern)
    s = glu.levelize(glu.detect_upward(fp))
    plans = glu.plan_schedule(s, glu.level_stats(fp, s), a.n, glu.ResourceModel())
    with pytest.raises(glu.ScheduleHazardError) as e:
        glu.factor_parallel(a, fp, s, plans, glu.FactorOptions(detect_races=True, deterministic=False))
    assert "writes element" in str(e.value) and e.value.hazards
    fp, s, plans = _analyze(a)
    lu, _ = glu.factor_parallel(a, fp, s, plans, glu.FactorOptions(detect_races=True, worker_count=2))
    assert glu.residual(a, lu) <= 1e-12


@pytest.fixture(scope="module")
def cfg2():
    from paper_1908_00204_b200 import synthetic

    a = synthetic.make("cfg2")
    fp, s, plans = _analyze(a, glu.B200_RESOURCE)
    return a, fp, s, plans


def _oracle_values(a, fp, s, deterministic):
    pat = orc.Pattern.from_fp(fp)
    v, bad = orc.scatter(pat, a.col_ptr, a.row_idx, a.values)
    assert bad == -1
    lp = np.concatenate([[0], np.cumsum([len(c) for c in s.levels])])
    caps = np.ones(len(s.levels), dtype=np.int64)
    assert orc.factor_parallel(pat, v, lp, np.concatenate(s.levels), caps, deterministic) == -1
    return v


@pytest.mark.parametrize("det", [True, False])
def test_cfg2_full_size_bitwise_vs_oracle(cfg2, det):
    a, fp, s, plans = cfg2
    lu, _ = glu.factor_parallel(a, fp, s, plans, glu.FactorOptions(deterministic=det))
    ref = _oracle_values(a, fp, s, det)
    assert np.array_equal(lu.values, ref)


def test_cfg2_refactorize_and_solve(cfg2):
    from paper_1908_00204_b200 import synthetic

    a, fp, s, plans = cfg2
    lu, _ = glu.factor_parallel(a, fp, s, plans, glu.FactorOptions(deterministic=False))
    a2 = glu.CscMatrix(a.n, a.col_ptr, a.row_idx, synthetic.perturb_values(a, 1000))
    lu2 = glu.refactorize(lu, a2, s, glu.FactorOptions(deterministic=False))
    assert np.array_equal(lu2.values, _oracle_values(a2, fp, s, False))
    b = np.random.default_rng(3).standard_normal(a.n)
    x = glu.solve(lu2, b)
    pat = orc.Pattern.from_fp(fp)
    xr, bad = orc.upper_solve(pat, lu2.values, orc.lower_solve(pat, lu2.values, b))
    assert bad == -1 and np.array_equal(x, xr)
    import scipy.sparse as sp

    A = sp.csc_matrix((a2.values, a2.row_idx, a2.col_ptr), shape=(a.n, a.n))
    assert np.linalg.norm(A @ x - b) / np.linalg.norm(b) <= 1e-10


def test_device_api_matches_host_api(cfg2):
    import torch

    a, fp, s, plans = cfg2
    fz = glu.get_factorizer(fp, s.level_of, 1)
    fz.set_input(a.col_ptr, a.row_idx)
    host, rc = fz.factor_host(a.values, 1e-14)
    assert rc == -1
    dev = torch.device("cuda")
    a_d = torch.from_numpy(a.values).to(dev)
    v_d = torch.empty(fp.nnz, dtype=torch.float64, device=dev)
    for _ in range(2):  # repeatable
        fz.scatter_device(a_d, v_d)
        assert fz.factor_device(v_d, 1e-14) == -1
        assert np.array_equal(v_d.cpu().numpy(), host)


def _cfg1_batch():
    from paper_1908_00204_b200 import synthetic

    a = synthetic.make("cfg1")
    fp, s, plans = _analyze(a)
    vals = np.stack([synthetic.perturb_values(a, 1000 + b) for b in range(5)])
    vals[2] = 0.0  # singular set: pivot breakdown inside the batch
    return a, fp, s, plans, vals


@pytest.mark.parametrize("det", [True, False])
def test_refactorize_batch_bitwise_per_set(det):
    a, fp, s, plans, vals = _cfg1_batch()
    lu, _ = glu.factor_parallel(a, fp, s, plans, glu.FactorOptions(deterministic=det))
    out, fails = glu.refactorize_batch(lu, a, vals, s, glu.FactorOptions(deterministic=det))
    pat = orc.Pattern.from_fp(fp)
    lp = np.concatenate([[0], np.cumsum([len(c) for c in s.levels])])
    for b in range(len(vals)):
        ref, bad = orc.scatter(pat, a.col_ptr, a.row_idx, vals[b])
        rc = orc.factor_parallel(pat, ref, lp, np.concatenate(s.levels),
                                 np.ones(len(lp) - 1, np.int64), det)
        assert int(fails[b]) == rc
        if rc == -1:
            assert np.array_equal(out[b], ref)
    assert fails[2] >= 0


@pytest.mark.parametrize("tail", [True, False])
def test_batch_device_matches_single_calls(tail):
    import torch

    a, fp, s, plans, vals = _cfg1_batch()
    fz = glu.get_factorizer(fp, s.level_of, 1, tail=tail)
    fz.set_input(a.col_ptr, a.row_idx)
    dev = torch.device("cuda")
    v = torch.empty((len(vals), fp.nnz), dtype=torch.float64, device=dev)
    for b in range(len(vals)):
        fz.scatter_device(torch.from_numpy(vals[b]).to(dev), v[b])
    fails = fz.factor_batch_device(v, 1e-14)
    ref = glu.get_factorizer(fp, s.level_of, 1)
    ref.set_input(a.col_ptr, a.row_idx)
    for b in range(len(vals)):
        single, rc = ref.factor_host(vals[b], 1e-14)
        assert int(fails[b]) == rc
        if rc == -1:
            assert np.array_equal(v[b].cpu().numpy(), single)


def test_cfg2_batched_launch_bitwise():
    """Eight value sets in one tail-less launch == eight single factorizations."""
    import torch
    from paper_1908_00204_b200 import synthetic

    a = synthetic.make("cfg2")
    fp, s, plans = _analyze(a, glu.B200_RESOURCE)
    vals = np.stack([synthetic.perturb_values(a, 2000 + b) for b in range(8)])
    out, fails = glu.refactorize_batch(glu.LuFactors(fp, np.zeros(fp.nnz)), a, vals, s,
                                       glu.FactorOptions(deterministic=False))
    assert np.all(fails == -1)
    for b in (0, 5, 7):
        assert np.array_equal(out[b], _oracle_values(glu.CscMatrix(a.n, a.col_ptr, a.row_idx, vals[b]),
                                                     fp, s, False))


def test_solve_many_matches_single_solves():
    from paper_1908_00204_b200 import synthetic

    a = synthetic.make("cfg1")
    fp, s, plans = _analyze(a)
    lu, _ = glu.factor_parallel(a, fp, s, plans, glu.FactorOptions())
    B = np.random.default_rng(7).standard_normal((a.n, 5))
    B[:, 3] = 0.0
    X = glu.solve_many(lu, B)
    for j in range(B.shape[1]):
        assert np.array_equal(X[:, j], glu.solve(lu, B[:, j]))


def _solve_factorizer(lu):
    return glu.get_factorizer(lu.pattern, glu.numeric._relaxed_levels(lu.pattern), 0)


def test_solve_entry_points_interleaved_bitwise():
    """Every solve entry point, interleaved in an order that exercises the
    dataflow solve's sentinel buffer hand-over (L-only leaves it via a move,
    U-only enters it via one); the removed level-synchronous kernel's option
    is refused."""
    from paper_1908_00204_b200 import synthetic

    a = synthetic.make("cfg1")
    fp, s, plans = _analyze(a)
    lu, _ = glu.factor_parallel(a, fp, s, plans, glu.FactorOptions())
    fz = _solve_factorizer(lu)
    with pytest.raises(glu.numeric._lib.GluError):
        fz.set_option(9, 1)
    fz.set_option(9, 0)
    pat = orc.Pattern.from_fp(fp)
    rng = np.random.default_rng(11)
    for step in range(3):
        b = rng.standard_normal(a.n)
        b[rng.integers(0, a.n, 50)] = 0.0
        yr = orc.lower_solve(pat, lu.values, b)
        xr, bad = orc.upper_solve(pat, lu.values, yr)
        assert bad == -1
        assert np.array_equal(glu.lower_solve(lu, b), yr), step
        assert np.array_equal(glu.solve(lu, b), xr), step
        assert np.array_equal(glu.upper_solve(lu, yr), xr), step
        B = np.stack([b, -b, np.zeros(a.n)], axis=1)
        X = glu.solve_many(lu, B)
        assert np.array_equal(X[:, 0], xr) and np.array_equal(X[:, 1], glu.solve(lu, -b))
        assert not X[:, 2].any()


def test_solve_rhs_carrying_the_sentinel_pattern():
    """The dataflow solve marks unfinished unknowns with one signalling-NaN
    bit pattern; an input carrying exactly that pattern must neither hang nor
    poison the next solve (it comes back quieted, still a NaN)."""
    a = glu.to_csc(glu.Triplets(3, 3, [0, 1, 2, 1], [0, 1, 2, 0], [2.0, 4.0, 8.0, 1.0]))
    fp = glu.symbolic_fillin(a.pattern)
    s = glu.levelize(glu.detect_relaxed(fp))
    plans = glu.plan_schedule(s, glu.level_stats(fp, s), a.n, glu.ResourceModel())
    lu, _ = glu.factor_parallel(a, fp, s, plans, glu.FactorOptions())
    b = np.array([0.0, 1.0, 1.0])
    b.view(np.uint64)[0] = np.uint64(0x7FF4DEAD5EB17A11)
    y = glu.lower_solve(lu, b)
    assert np.isnan(y[0]) and np.isnan(y[1]) and y[2] == 1.0
    x = glu.solve(lu, np.array([2.0, 5.0, 8.0]))
    assert np.array_equal(x, [1.0, 1.0, 1.0])


@pytest.mark.parametrize("multi", [1, 0])  # 1: lanes over right-hand sides, 0: one warp each
def test_solve_multi_parts_and_groups(multi):
    """k > 32 right-hand sides (two lane groups, a ragged last one) through
    glu_solve_multi_device for L then U, L only and U only, each column
    bitwise the oracle's single solve."""
    import ctypes

    import torch
    from paper_1908_00204_b200 import _lib, synthetic

    a = synthetic.make("cfg1")
    fp, s, plans = _analyze(a)
    lu, _ = glu.factor_parallel(a, fp, s, plans, glu.FactorOptions())
    fz = _solve_factorizer(lu)
    fz.set_option(11, multi)
    pat = orc.Pattern.from_fp(fp)
    k, ld = 41, a.n + 7
    B = np.random.default_rng(5).standard_normal((k, a.n))
    B[3] = 0.0
    Y = np.stack([orc.lower_solve(pat, lu.values, b) for b in B])
    X = np.stack([orc.upper_solve(pat, lu.values, y)[0] for y in Y])
    dev = torch.device("cuda", 0)
    lu_d = torch.from_numpy(lu.values).to(dev)
    try:
        for part, src, want in ((0, B, X), (1, B, Y), (2, Y, X), (0, B, X)):
            buf = torch.full((k, ld), 7.0, dtype=torch.float64, device=dev)
            buf[:, : a.n] = torch.from_numpy(src).to(dev)
            st = torch.cuda.current_stream()
            rc = _lib.lib.glu_solve_multi_device(fz.handle, glu.numeric._dptr(lu_d),
                                                 glu.numeric._dptr(buf), k, ld, part,
                                                 ctypes.c_void_p(st.cuda_stream))
            assert rc == -1, _lib.lib.glu_last_error()
            out = buf.cpu().numpy()
            assert np.array_equal(out[:, : a.n], want), part
            assert (out[:, a.n:] == 7.0).all()  # padding untouched
    finally:
        fz.set_option(11, 1)


@pytest.mark.parametrize("cfg", ["cfg3", "g200"])
@pytest.mark.parametrize("det", [True, False])
def test_full_size_bitwise_vs_oracle(cfg, det):
    """cfg3 (the deep, stream-mode schedule: 680k columns, 912 levels) and a
    G3-family grid (wide levels, deep hub items, the cluster dense tail) at
    full size, both contracts, against the C restatement of the reference."""
    from paper_1908_00204_b200 import synthetic

    a = synthetic.make(cfg) if cfg in synthetic.CONFIGS else synthetic.grid5(200, seed=0)
    fp, s, plans = _analyze(a, glu.B200_RESOURCE)
    lu, _ = glu.factor_parallel(a, fp, s, plans, glu.FactorOptions(deterministic=det))
    assert np.array_equal(lu.values, _oracle_values(a, fp, s, det))
    b = np.random.default_rng(1).standard_normal(a.n)
    pat = orc.Pattern.from_fp(fp)
    xr, bad = orc.upper_solve(pat, lu.values, orc.lower_solve(pat, lu.values, b))
    assert bad == -1 and np.array_equal(glu.solve(lu, b), xr)


def test_one_by_one():
    a = glu.to_csc(glu.Triplets(1, 1, [0], [0], [5.0]))
    fp, s, plans = _analyze(a)
    for det in (True, False):
        lu, _ = glu.factor_parallel(a, fp, s, plans, glu.FactorOptions(deterministic=det))
        assert lu.values.tolist() == [5.0]
    assert glu.solve(lu, np.array([10.0])).tolist() == [2.0]
    z = glu.to_csc(glu.Triplets(1, 1, [0], [0], [0.0]))
    with pytest.raises(glu.PivotError) as e:
        glu.factor_parallel(z, fp, s, plans, glu.FactorOptions())
    assert e.value.column == 0


@pytest.mark.parametrize("det", [True, False])
def test_pivot_breakdown_inside_cfg1_matches_oracle(det):
    """Shrink two diagonals of cfg1 (a low column in level 10, a high one in
    level 0) and raise the relative pivot threshold so both break down: the
    reported column is the oracle's for each path's order -- the earliest
    level's lowest column for factor_parallel (1483 here), the lowest column
    for the sequential paths (1414)."""
    from paper_1908_00204_b200 import synthetic

    a0 = synthetic.make("cfg1")
    fp, s, plans = _analyze(a0)
    cols = np.repeat(np.arange(a0.n), np.diff(a0.col_ptr))
    lv = np.asarray(s.level_of)
    lo = int(np.nonzero(lv >= 10)[0].min())  # a low column in a late level
    hi = int(np.nonzero(lv == 0)[0].max())   # a high column in level 0
    assert lo < hi
    vals = a0.values.copy()
    for c in (lo, hi):
        vals[(a0.row_idx == c) & (cols == c)] *= 0.01
    a = glu.CscMatrix(a0.n, a0.col_ptr, a0.row_idx, vals)
    th = 0.5
    pat = orc.Pattern.from_fp(fp)
    lp = np.concatenate([[0], np.cumsum([len(c) for c in s.levels])])
    v, _ = orc.scatter(pat, a.col_ptr, a.row_idx, a.values)
    want = orc.factor_parallel(pat, v, lp, np.concatenate(s.levels),
                               np.ones(len(s.levels), dtype=np.int64), det, th)
    v, _ = orc.scatter(pat, a.col_ptr, a.row_idx, a.values)
    want_seq = orc.factor_left_looking(pat, v, th)
    assert want == hi and want_seq == lo  # the orders differ on this input
    with pytest.raises(glu.PivotError) as e:
        glu.factor_parallel(a, fp, s, plans,
                            glu.FactorOptions(deterministic=det, zero_pivot_threshold=th))
    assert e.value.column == want
    for fn in (glu.factor_left_looking, glu.factor_right_looking_seq):
        with pytest.raises(glu.PivotError) as e:
            fn(a, fp, glu.FactorOptions(zero_pivot_threshold=th))
        assert e.value.column == want_seq


def test_solve_batch_per_set_bitwise():
    """refactorize_batch -> solve_batch (the Newton-loop pair): every set's
    solution is bitwise the oracle's solve with that set's factors; a set
    with an exactly zero diagonal reports the column upper_solve raises."""
    from paper_1908_00204_b200 import synthetic

    a = synthetic.make("cfg1")
    fp, s, plans = _analyze(a)
    lu, _ = glu.factor_parallel(a, fp, s, plans, glu.FactorOptions())
    nb = 6
    vals = np.stack([synthetic.perturb_values(a, 100 + k) for k in range(nb)])
    L, st = glu.refactorize_batch(lu, a, vals)
    assert (st == -1).all()
    L = L.copy()
    bad_col = int(np.asarray(s.level_of).argmax())
    L[4, fp.diag_pos[bad_col]] = 0.0  # set 4: a zero diagonal
    B = np.random.default_rng(9).standard_normal((nb, a.n))
    B[2] = 0.0
    X, status = glu.solve_batch(lu, L, B)
    pat = orc.Pattern.from_fp(fp)
    for k in range(nb):
        y = orc.lower_solve(pat, L[k], B[k])
        xr, bad = orc.upper_solve(pat, L[k], y)
        assert status[k] == bad, k
        if bad == -1:
            assert np.array_equal(X[k], xr), k
    assert status[4] >= 0 and (status[[0, 1, 2, 3, 5]] == -1).all()


def test_batched_tail_failure_in_one_set():
    """A batched launch whose dense tail fails for one value set only: that
    set reports the single launch's failing column (inside the tail), the
    other sets' factors are bitwise the single launches'."""
    import torch
    from paper_1908_00204_b200 import synthetic

    a = synthetic.make("cfg1")
    fp, s, plans = _analyze(a)
    cols = np.repeat(np.arange(a.n), np.diff(a.col_ptr))
    vals = np.stack([synthetic.perturb_values(a, 2000 + b) for b in range(6)])
    last = a.n - 1
    th = 1e-14
    ref = glu.get_factorizer(fp, s.level_of, 1)
    ref.set_input(a.col_ptr, a.row_idx)
    lu3, rc3 = ref.factor_host(vals[3], th)
    assert rc3 == -1
    # subtract set 3's final pivot of the last (tail) column from its A entry:
    # the recomputed pivot cancels to rounding level and breaks down there
    vals[3][(a.row_idx == last) & (cols == last)] -= lu3[fp.diag_pos[last]]
    fz = glu.get_factorizer(fp, s.level_of, 1, tail=False)
    assert fz.plan_info["tail_t0"] < a.n  # the batch plan has a dense tail
    fz.set_input(a.col_ptr, a.row_idx)
    dev = torch.device("cuda")
    v = torch.empty((len(vals), fp.nnz), dtype=torch.float64, device=dev)
    for b in range(len(vals)):
        fz.scatter_device(torch.from_numpy(vals[b]).to(dev), v[b])
    fails = fz.factor_batch_device(v, th)
    for b in range(len(vals)):
        single, rc = ref.factor_host(vals[b], th)
        assert int(fails[b]) == rc, b
        if rc == -1:
            assert np.array_equal(v[b].cpu().numpy(), single), b
    assert int(fails[3]) >= fz.plan_info["tail_t0"]
    assert all(int(fails[b]) == -1 for b in (0, 1, 2, 4, 5))


def test_single_precision_inputs():
    """fp32 values (the reference's single precision, tests/test_numeric.py:
    203-210): factored in fp64 on the device, returned as fp32 factors within
    the reference's fp32 residual bound; solves return fp32."""
    from conftest import random_dd

    a = random_dd(np.random.default_rng(11), 40, 0.1)
    a32 = glu.CscMatrix(a.n, a.col_ptr, a.row_idx, a.values.astype(np.float32))
    fp, s, plans = _analyze(a32)
    lu, _ = glu.factor_parallel(a32, fp, s, plans, glu.FactorOptions(worker_count=2))
    assert lu.values.dtype == np.float32
    assert glu.residual(a32, lu) <= 1e-5
    lu64 = glu.factor_left_looking(glu.CscMatrix(a.n, a.col_ptr, a.row_idx,
                                                 a.values.astype(np.float32).astype(np.float64)), fp)
    assert np.array_equal(lu.values, lu64.values.astype(np.float32))
    x = glu.solve(lu, np.ones(a.n, dtype=np.float32))
    assert x.dtype == np.float32 and np.all(np.isfinite(x))


def test_level_times_opt_in(monkeypatch):
    """FactorStats.level_times: one entry per caller level; GPU completion
    times only with GLU_LEVEL_TIMES=1 (zeros otherwise), the values bitwise
    the same either way."""
    g = load_golden("cfg1")
    a = csc_from_golden(g)
    fp = glu.symbolic_fillin(a.pattern)
    s = glu.levelize(glu.detect_relaxed(fp))
    plans = glu.plan_schedule(s, glu.level_stats(fp, s), a.n, glu.B200_RESOURCE)
    monkeypatch.setenv("GLU_LEVEL_TIMES", "0")
    lu0, st0 = glu.factor_parallel(a, fp, s, plans, glu.FactorOptions())
    assert st0.level_times == [0.0] * s.level_count
    monkeypatch.setenv("GLU_LEVEL_TIMES", "1")
    lu1, st1 = glu.factor_parallel(a, fp, s, plans, glu.FactorOptions())
    assert len(st1.level_times) == s.level_count and sum(st1.level_times) > 0.0
    assert np.array_equal(lu0.values, lu1.values)


def test_pinned_results_own_their_buffers(monkeypatch):
    """Results in page-locked pool buffers (numeric._PinnedPool): a kept
    result is never overwritten by a later factorization, a dropped one's
    buffer is reused, and every result is bitwise the oracle's."""
    import gc

    from paper_1908_00204_b200 import numeric, synthetic

    monkeypatch.setattr(numeric, "_PINNED_MIN", 0)
    a = synthetic.make("cfg1")
    fp, s, plans = _analyze(a)
    pat = orc.Pattern.from_fp(fp)
    opts = glu.FactorOptions(deterministic=True)

    def oracle(vals):
        v, bad = orc.scatter(pat, a.col_ptr, a.row_idx, vals)
        assert bad == -1 and orc.factor_left_looking(pat, v, opts.zero_pivot_threshold) == -1
        return v

    lu1, _ = glu.factor_parallel(a, fp, s, plans, opts)
    keep = lu1.values.copy()
    assert np.array_equal(keep, oracle(a.values))
    a2 = glu.CscMatrix(a.n, a.col_ptr, a.row_idx, synthetic.perturb_values(a, seed=3))
    lu2, _ = glu.factor_parallel(a2, fp, s, plans, opts)
    assert np.array_equal(lu1.values, keep)  # not aliased by the second result
    assert np.array_equal(lu2.values, oracle(a2.values))
    addr2 = lu2.values.ctypes.data
    del lu2
    gc.collect()
    lu3, _ = glu.factor_parallel(a, fp, s, plans, opts)
    assert lu3.values.ctypes.data == addr2  # the dropped buffer came back from the pool
    assert np.array_equal(lu3.values, keep)
    assert lu3.values.flags.writeable and lu3.values.flags.c_contiguous
