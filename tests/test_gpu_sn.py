"""B200 parity of the supernodal engine (glu_snode.cu) and of caller
schedules other than the relaxed one, through the C ABI, against the
reference's goldens and the CPU oracle (bit for bit, contract A)."""

from __future__ import annotations

import numpy as np
import pytest

import paper_1908_00204_b200 as glu
from paper_1908_00204_b200 import numeric, synthetic
from conftest import csc_from_golden, golden_cases, load_golden
from oracle import oracle as orc

pytestmark = pytest.mark.gpu


def _sn_factor(a, fp, thresh=1e-14, by_column=True, level_of=None):
    lv = numeric._relaxed_levels(fp)
    fz = numeric.get_factorizer(fp, lv, glu.numeric._lib.CONTRACT_A, engine="sn")
    assert fz.engine == "sn"
    with fz._lock:
        fz.set_input(a.col_ptr, a.row_idx)
        fz.set_fail_levels(lv if level_of is None else level_of)
        fz.set_option(2, 1 if by_column else 0)
        fz.set_option(1, 0)
        vals, rc = fz.factor_host(a.values, thresh)
    return vals, rc, fz


def _oracle_a(fp, a):
    pat = orc.Pattern.from_fp(fp)
    v, bad = orc.scatter(pat, a.col_ptr, a.row_idx, a.values)
    assert bad == -1
    return v, orc.factor_left_looking(pat, v, 1e-14)


@pytest.mark.parametrize("name", golden_cases())
def test_sn_goldens_bitwise(name):
    g = load_golden(name)
    a = csc_from_golden(g)
    fp = glu.symbolic_fillin(a.pattern)
    vals, rc, _ = _sn_factor(a, fp, float(g["thresh"]))
    if int(g["fail_a"]) >= 0:
        assert rc == int(g["fail_a"])
    else:
        assert rc == -1 and np.array_equal(vals, g["lu_a"]), name


@pytest.mark.parametrize("k", [24, 64, 150])
def test_sn_grid_bitwise(k):
    a = synthetic.grid5(k, seed=k)
    fp = glu.symbolic_fillin(a.pattern)
    ref, err = _oracle_a(fp, a)
    vals, rc, fz = _sn_factor(a, fp)
    assert err == -1 and rc == -1
    assert np.array_equal(vals, ref)
    # a second call on the resident plan (refactorization) is identical
    vals2, rc2, _ = _sn_factor(a, fp)
    assert rc2 == -1 and np.array_equal(vals2, ref)


def test_sn_cfg1_and_unsymmetric_bitwise():
    from conftest import random_dd

    for a in (synthetic.make("cfg1"), random_dd(np.random.default_rng(5), 400, 0.01)):
        fp = glu.symbolic_fillin(a.pattern)
        ref, err = _oracle_a(fp, a)
        vals, rc, _ = _sn_factor(a, fp)
        assert err == -1 and rc == -1 and np.array_equal(vals, ref)


def test_sn_pivot_failure_column():
    """A zero pivot inside a wide supernode is reported at the reference's
    column (first failing column), the later garbage notwithstanding."""
    a = synthetic.grid5(40, seed=1)
    fp = glu.symbolic_fillin(a.pattern)
    v = a.values.copy()
    cols = np.repeat(np.arange(a.n), np.diff(a.col_ptr))
    target = a.n - 30  # inside the top separator
    v[(cols == target) & (a.row_idx == target)] = 0.0
    # make it exactly singular after elimination: a zero column
    v[cols == target] = 0.0
    bad = glu.CscMatrix(a.n, a.col_ptr, a.row_idx, v)
    pat = orc.Pattern.from_fp(fp)
    ref, _ = orc.scatter(pat, bad.col_ptr, bad.row_idx, bad.values)
    err = orc.factor_left_looking(pat, ref, 1e-14)
    assert err >= 0
    _, rc, _ = _sn_factor(bad, fp)
    assert rc == err


def test_sn_g200_full_size_bitwise():
    a = synthetic.grid5(200, seed=0)
    fp = glu.symbolic_fillin(a.pattern)
    ref, err = _oracle_a(fp, a)
    vals, rc, fz = _sn_factor(a, fp)
    assert err == -1 and rc == -1 and np.array_equal(vals, ref)
    assert fz.sn_info["macs"] == numeric.pattern_flops(fp)[0]


def test_sn_g400_full_size_bitwise():
    a = synthetic.make("g400")
    fp = glu.symbolic_fillin(a.pattern)
    ref, err = _oracle_a(fp, a)
    vals, rc, _ = _sn_factor(a, fp)
    assert err == -1 and rc == -1 and np.array_equal(vals, ref)


def test_sn_batch_sets_bitwise():
    """refactorize_batch through the supernodal engine (one launch per set):
    every set bitwise, a singular set reported at its own column."""
    import os

    old = os.environ.get("GLU_ENGINE")
    os.environ["GLU_ENGINE"] = "sn"
    try:
        a = synthetic.grid5(40, seed=3)
        fp = glu.symbolic_fillin(a.pattern)
        lu = glu.factor_left_looking(a, fp)
        sets = np.stack([synthetic.perturb_values(a, 50 + b) for b in range(3)])
        sets[1] = 0.0
        vals, st = glu.refactorize_batch(lu, a, sets)
        pat = orc.Pattern.from_fp(fp)
        for b in range(3):
            v, _ = orc.scatter(pat, a.col_ptr, a.row_idx, sets[b])
            err = orc.factor_left_looking(pat, v)
            assert st[b] == err
            if err == -1:
                assert np.array_equal(vals[b], v)
    finally:
        if old is None:
            os.environ.pop("GLU_ENGINE", None)
        else:
            os.environ["GLU_ENGINE"] = old


def test_sn_public_api_engine_switch(monkeypatch):
    """GLU_ENGINE=sn routes the reference API (left-looking, factor_parallel
    deterministic, refactorize) through the supernodal engine."""
    monkeypatch.setenv("GLU_ENGINE", "sn")
    a = synthetic.grid5(48, seed=2)
    fp = glu.symbolic_fillin(a.pattern)
    s = glu.levelize(glu.detect_relaxed(fp))
    plans = glu.plan_schedule(s, glu.level_stats(fp, s), a.n, glu.B200_RESOURCE)
    ref, _ = _oracle_a(fp, a)
    lu = glu.factor_left_looking(a, fp)
    assert np.array_equal(lu.values, ref)
    lu2, st = glu.factor_parallel(a, fp, s, plans, glu.FactorOptions(worker_count=4))
    assert np.array_equal(lu2.values, ref) and len(st.level_times) == s.level_count
    assert np.array_equal(glu.refactorize(lu, a).values, ref)
    x = glu.solve(lu, np.ones(a.n))
    assert glu.numeric.residual(a, lu) < 1e-12 and np.all(np.isfinite(x))


@pytest.mark.parametrize("name", ["conflict8", "random_dd_s2_n80", "random_dd_s12_n500", "cfg1",
                                  "singular_2x2", "block_arrow_4x24"])
@pytest.mark.parametrize("workers", [1, 2])
def test_upward_schedule_bitwise(name, workers):
    """factor_parallel under levelize(detect_upward(fp)): deterministic and
    atomic mode against the oracle's factor_parallel on the same schedule."""
    g = load_golden(name)
    a = csc_from_golden(g)
    fp = glu.symbolic_fillin(a.pattern)
    s = glu.levelize(glu.detect_upward(fp))
    plans = glu.plan_schedule(s, glu.level_stats(fp, s), a.n, glu.ResourceModel())
    pat = orc.Pattern.from_fp(fp)
    lp = np.concatenate([[0], np.cumsum([len(c) for c in s.levels])]).astype(np.int64)
    lc = np.concatenate(s.levels).astype(np.int64)
    thr = float(g["thresh"])
    for det in (True, False):
        ref, _ = orc.scatter(pat, a.col_ptr, a.row_idx, a.values)
        err = orc.factor_parallel(pat, ref, lp, lc, np.full(len(lp) - 1, workers, np.int64), det, thr)
        opts = glu.FactorOptions(deterministic=det, worker_count=workers, zero_pivot_threshold=thr)
        if err >= 0:
            with pytest.raises(glu.PivotError) as e:
                glu.factor_parallel(a, fp, s, plans, opts)
            assert e.value.column == err
        else:
            lu, st = glu.factor_parallel(a, fp, s, plans, opts)
            assert np.array_equal(lu.values, ref), (name, det)
            assert len(st.level_times) == s.level_count


def test_cli_upward_checksum(tmp_path, capsys):
    """levlu factor conflict8.mtx --deps upward --parallel --allow-unsafe
    prints the reference's checksum (tests/test_cli.py:140-154)."""
    from paper_1908_00204_b200 import cli
    from test_cli import _write_mtx

    mtx = _write_mtx(tmp_path / "conflict8.mtx", load_golden("conflict8"))
    for extra in ([], ["--threads", "2"]):
        assert cli.main(["factor", mtx, "--deps", "upward", "--parallel", "--allow-unsafe"] + extra) == 0
        assert "checksum cb2c3e22567ad657" in capsys.readouterr().out
