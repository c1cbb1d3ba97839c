"""Host analysis of the B200 path (native C++) is bit-exact vs the reference."""

from __future__ import annotations

import warnings

import numpy as np
import pytest

import paper_1908_00204_b200 as glu
from conftest import GOLDEN, csc_from_golden, load_golden, pattern_from_golden, random_dd
from oracle import oracle as orc


def test_pattern_and_schedule_match_reference(golden):
    name, g = golden
    a = csc_from_golden(g)
    fp = glu.symbolic_fillin(a.pattern)
    assert np.array_equal(fp.full.col_ptr, g["fp_col_ptr"])
    assert np.array_equal(fp.full.row_idx, g["fp_row_idx"])
    assert np.array_equal(fp.diag_pos, g["fp_diag_pos"])
    assert np.array_equal(fp.csr.row_ptr, g["csr_row_ptr"])
    assert np.array_equal(fp.csr.col_idx, g["csr_col_idx"])
    assert np.array_equal(fp.csr.csc_pos, g["csr_csc_pos"])
    assert fp.nz_before == int(g["nz_before"])
    gr = glu.detect_relaxed(fp)
    assert np.array_equal(gr.dep_ptr, g["relaxed_ptr"]) and np.array_equal(gr.dep_idx, g["relaxed_idx"])
    gu = glu.detect_upward(fp)
    assert np.array_equal(gu.dep_ptr, g["upward_ptr"]) and np.array_equal(gu.dep_idx, g["upward_idx"])
    s = glu.levelize(gr)
    assert np.array_equal(s.level_of, g["level_of"])
    assert np.array_equal(np.concatenate(s.levels), g["level_cols"])
    st = glu.level_stats(fp, s)
    assert st.sizes == g["stat_sizes"].tolist()
    assert st.max_subcolumns == g["stat_max_sub"].tolist()
    plans = glu.plan_schedule(s, st, a.n, glu.ResourceModel())
    assert [p.mode.value for p in plans] == g["modes_default"].tolist()
    assert [p.warps_per_column for p in plans] == g["wpb_default"].tolist()
    plans = glu.plan_schedule(s, glu.level_stats(fp, s), a.n, glu.B200_RESOURCE)
    assert [p.mode.value for p in plans] == g["modes_b200"].tolist()
    if "flop_count" in g:
        assert sum(glu.pattern_flops(fp)) == int(g["flop_count"])


@pytest.mark.parametrize("seed,n,density", [(21, 700, 0.004), (22, 1500, 0.002), (23, 3000, 0.0008)])
def test_analysis_matches_oracle_random(seed, n, density):
    a = random_dd(np.random.default_rng(seed), n, density)
    fp = glu.symbolic_fillin(a.pattern)
    pat = orc.symbolic_fillin(n, a.col_ptr, a.row_idx)
    assert np.array_equal(fp.full.row_idx, pat.row_idx)
    assert np.array_equal(fp.full.col_ptr, pat.col_ptr)
    assert np.array_equal(fp.csr.csc_pos, pat.csc_pos)
    gr = glu.detect_relaxed(fp)
    ptr, idx = orc.relaxed_deps(pat)
    assert np.array_equal(gr.dep_ptr, ptr) and np.array_equal(gr.dep_idx, idx)
    s = glu.levelize(gr)
    lv, lp, lc = orc.levelize(n, ptr, idx)
    assert np.array_equal(s.level_of, lv)


def test_synthetic_cfg1_analysis_matches_oracle():
    from paper_1908_00204_b200 import synthetic

    a = synthetic.make("cfg1")
    fp = glu.symbolic_fillin(a.pattern)
    pat = orc.symbolic_fillin(a.n, a.col_ptr, a.row_idx)
    assert np.array_equal(fp.full.row_idx, pat.row_idx)


def test_symbolic_errors():
    a = glu.CscMatrix(2, np.array([0, 1, 1]), np.array([0]), np.array([1.0]))
    with pytest.raises(glu.SymbolicError, match="structurally empty"):
        glu.symbolic_fillin(a.pattern)
    b = glu.to_csc(glu.Triplets(2, 2, [0, 0], [0, 1], [1.0, 1.0]))
    with pytest.raises(glu.SymbolicError, match="diagonal missing"):
        glu.symbolic_fillin(b.pattern, inject_diagonal=False)
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        fp = glu.symbolic_fillin(b.pattern)
    assert any("injected 1" in str(x.message) for x in w)
    assert fp.full.has_entry(1, 1)


def test_levelize_accepts_reference_style_graph():
    class G:  # duck-typed levlu.DependencyGraph
        n = 4
        deps = [np.array([], np.int64), np.array([0]), np.array([], np.int64), np.array([1, 2])]

    s = glu.levelize(G())
    assert [c.tolist() for c in s.levels] == [[0, 2], [1], [3]]


def test_hazards_on_upward_schedule_of_conflict8():
    """The reference's known hazard (tests/test_depgraph.py:129-137): writer 3,
    reader 5, element (5, 6) under the upward schedule; none under relaxed."""
    from conftest import load_golden

    a = csc_from_golden(load_golden("conflict8"))
    fp = glu.symbolic_fillin(a.pattern)
    hz = glu.find_hazards(fp, glu.levelize(glu.detect_upward(fp)))
    assert any(h.writer == 3 and h.reader == 5 and h.element == (5, 6) for h in hz)
    assert glu.find_hazards(fp, glu.levelize(glu.detect_relaxed(fp))) == []


DG_CASES = ["conflict8", "random_dd_s1_n40", "random_dd_s2_n80", "random_dd_s3_n120", "random_dd_s5_n100",
            "block_arrow_4x24", "banded_n200", "cfg1"]


def _dg_golden(name):
    with np.load(GOLDEN / "depgraph" / f"{name}.npz") as d:
        return {k: d[k] for k in d.files}


@pytest.mark.parametrize("name", DG_CASES)
def test_double_u_exact_and_hazards_match_reference(name):
    """detect_double_u_exact and simulate_hazards (levlu/depgraph.py:129-156,
    :173-205) against the reference's own outputs (tests/golden/make_depgraph.py)."""
    g = load_golden(name)
    d = _dg_golden(name)
    fp = glu.symbolic_fillin(csc_from_golden(g).pattern)
    ex = glu.detect_double_u_exact(fp)
    assert ex.method is glu.DetectMethod.DOUBLE_U_EXACT
    assert np.array_equal(ex.dep_ptr, d["exact_ptr"]) and np.array_equal(ex.dep_idx, d["exact_idx"])
    for sched, key in ((glu.levelize(glu.detect_upward(fp)), "hz_upward"),
                       (glu.levelize(glu.detect_relaxed(fp)), "hz_relaxed")):
        rep = glu.simulate_hazards(fp, sched)
        got = np.array([[h.level, h.writer, h.reader, h.element[0], h.element[1]] for h in rep.hazards],
                       dtype=np.int64).reshape(-1, 5)
        assert np.array_equal(got, d[key]), (name, key)
        assert len(rep) == len(d[key])


def test_dependency_graph_constructor_and_partition_check():
    """DependencyGraph(n, deps, method) as the reference's dataclass; a
    schedule that is not a partition is rejected like the reference."""
    g = glu.DependencyGraph(3, [np.array([], np.int64), np.array([0]), np.array([0, 1])],
                            glu.DetectMethod.RELAXED)
    assert g.edge_count == 3 and g.edge_set() == {(1, 0), (2, 0), (2, 1)}
    s = glu.levelize(g)
    assert [c.tolist() for c in s.levels] == [[0], [1], [2]]
    fp = glu.symbolic_fillin(csc_from_golden(load_golden("conflict8")).pattern)
    bad = glu.LevelSchedule([np.array([0, 1])], np.zeros(fp.n, np.int64))
    with pytest.raises(ValueError):
        glu.simulate_hazards(fp, bad)


def _digests():
    import json

    return json.loads((GOLDEN / "analysis_digests.json").read_text())


@pytest.mark.parametrize("name", ["cfg2", "cfg3", "cfg4"])
def test_analysis_bit_exact_at_config_scale(name):
    """The C++ analysis at the BASELINE configs' sizes against sha256 digests
    of the reference's own arrays (tests/golden/make_digests.py ran
    levlu.symbolic_fillin / detect_relaxed / levelize on the same seeded
    matrices; cfg4 took the reference 144 s)."""
    import hashlib

    from paper_1908_00204_b200 import synthetic

    want = _digests()[name]

    def dg(x):
        return hashlib.sha256(np.ascontiguousarray(x, dtype="<i8").tobytes()).hexdigest()

    a = synthetic.make(name)
    fp = glu.symbolic_fillin(a.pattern)
    assert fp.nnz == want["nnz"]
    assert dg(fp.full.col_ptr) == want["col_ptr"] and dg(fp.full.row_idx) == want["row_idx"]
    assert dg(fp.diag_pos) == want["diag_pos"] and dg(fp.csr.csc_pos) == want["csc_pos"]
    s = glu.levelize(glu.detect_relaxed(fp))
    assert s.level_count == want["levels"] and dg(s.level_of) == want["level_of"]
