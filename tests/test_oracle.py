"""Pin the CPU oracle (oracle/) to the reference's own outputs (tests/golden)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import pattern_from_golden
from oracle import oracle as orc


def _caps(g, workers):
    sizes = np.diff(g["level_ptr"])
    return orc.concurrency_caps([int(s) for s in sizes], workers, n=int(g["n"]))


def test_symbolic_matches_reference(golden):
    name, g = golden
    pat = orc.symbolic_fillin(int(g["n"]), g["a_col_ptr"], g["a_row_idx"])
    assert np.array_equal(pat.col_ptr, g["fp_col_ptr"])
    assert np.array_equal(pat.row_idx, g["fp_row_idx"])
    assert np.array_equal(pat.diag_pos, g["fp_diag_pos"])
    assert np.array_equal(pat.row_ptr, g["csr_row_ptr"])
    assert np.array_equal(pat.col_idx, g["csr_col_idx"])
    assert np.array_equal(pat.csc_pos, g["csr_csc_pos"])


def test_dependencies_and_levels_match_reference(golden):
    name, g = golden
    pat = pattern_from_golden(g)
    ptr, idx = orc.relaxed_deps(pat)
    assert np.array_equal(ptr, g["relaxed_ptr"]) and np.array_equal(idx, g["relaxed_idx"])
    lv, lp, lc = orc.levelize(pat.n, ptr, idx)
    assert np.array_equal(lv, g["level_of"])
    assert np.array_equal(lp, g["level_ptr"]) and np.array_equal(lc, g["level_cols"])


def _scattered(g, pat):
    v, bad = orc.scatter(pat, g["a_col_ptr"], g["a_row_idx"], g["a_values"])
    assert bad == -1
    return v


def test_left_looking_matches_reference(golden):
    name, g = golden
    pat = pattern_from_golden(g)
    v = _scattered(g, pat)
    err = orc.factor_left_looking(pat, v, float(g["thresh"]))
    if int(g["fail_a"]) >= 0:
        assert err == int(g["fail_a"])
    else:
        assert err == -1
        assert np.array_equal(v, g["lu_a"])


def test_right_looking_seq_matches_reference(golden):
    name, g = golden
    pat = pattern_from_golden(g)
    v = _scattered(g, pat)
    err = orc.factor_right_looking_seq(pat, v, float(g["thresh"]))
    if int(g["fail_rl"]) >= 0:
        assert err == int(g["fail_rl"])
    else:
        assert err == -1 and np.array_equal(v, g["lu_rl"])


@pytest.mark.parametrize("workers", [1, 2, 8])
@pytest.mark.parametrize("deterministic", [True, False])
def test_factor_parallel_matches_reference(golden, workers, deterministic):
    """Contract A (det) and contract B (atomic) are worker-count invariant."""
    name, g = golden
    pat = pattern_from_golden(g)
    v = _scattered(g, pat)
    err = orc.factor_parallel(pat, v, g["level_ptr"], g["level_cols"], _caps(g, workers),
                              deterministic, float(g["thresh"]))
    tag = "det" if deterministic else "b"
    if int(g[f"fail_{tag}"]) >= 0:
        assert err == int(g[f"fail_{tag}"])
    else:
        assert err == -1 and np.array_equal(v, g[f"lu_{tag}"])


def test_solves_match_reference(golden):
    name, g = golden
    if "rhs" not in g:
        pytest.skip("factorization fails for this case")
    pat = pattern_from_golden(g)
    y = orc.lower_solve(pat, g["lu_a"], g["rhs"])
    assert np.array_equal(y, g["y_lower"])
    x, bad = orc.upper_solve(pat, g["lu_a"], y)
    assert bad == -1 and np.array_equal(x, g["x_upper"])


def test_flop_count_matches_reference(golden):
    name, g = golden
    if "flop_count" not in g:
        pytest.skip("no successful factor_parallel")
    macs, total = orc.pattern_flops(pattern_from_golden(g))
    assert total == int(g["flop_count"])


def test_known_answers():
    """Hand values from the reference tests (tests/test_numeric.py:20-31,
    SURVEY.md 8(c) conflict8 values)."""
    from conftest import load_golden

    g = load_golden("two_by_two")
    assert g["lu_a"].tolist() == [4.0, 1.5, 3.0, -1.5]
    assert g["y_lower"].tolist()[0] == g["rhs"][0]
    c8 = load_golden("conflict8")
    assert c8["lu_a"].tolist() == [8.0, 0.125, 0.5, 7.9375, 8.0, 8.0, -0.0625, 0.03125, -1.0,
                                   8.0, 8.0, -0.09375, 1.25, 1.078125, 8.0, 0.07025146484375,
                                   0.75, 1.0, 7.92974853515625]
    lp, lc = c8["level_ptr"], c8["level_cols"]
    assert [lc[lp[i]:lp[i + 1]].tolist() for i in range(len(lp) - 1)] == [[0, 2, 3, 4], [1, 5], [6], [7]]
    assert load_golden("singular_2x2")["fail_a"] == 1


def test_oracle_analysis_matches_reference(golden):
    """The oracle's analysis restatement (the reference arm of bench.py runs
    it instead of the product's C++): symbolic fill-in, relaxed deps and
    levels bit-exact against the reference's own outputs."""
    name, g = golden
    n = int(g["n"])
    pat = orc.symbolic_fillin(n, g["a_col_ptr"], g["a_row_idx"])
    assert np.array_equal(pat.col_ptr, g["fp_col_ptr"]) and np.array_equal(pat.row_idx, g["fp_row_idx"])
    assert np.array_equal(pat.diag_pos, g["fp_diag_pos"])
    ptr, idx = orc.relaxed_deps(pat)
    assert np.array_equal(ptr, g["relaxed_ptr"]) and np.array_equal(idx, g["relaxed_idx"])
    level_of, lp, lc = orc.levelize(n, ptr, idx)
    assert np.array_equal(level_of, g["level_of"])
    assert np.array_equal(lp, g["level_ptr"]) and np.array_equal(lc, g["level_cols"])


def test_oracle_analysis_matches_product_at_scale():
    """Same arrays as the product's C++ analysis on a 100k-row grid."""
    import paper_1908_00204_b200 as glu
    from paper_1908_00204_b200 import synthetic

    a = synthetic.grid5(150, drop=0.1, seed=4)
    pat = orc.symbolic_fillin(a.n, a.col_ptr, a.row_idx)
    fp = glu.symbolic_fillin(a.pattern)
    assert np.array_equal(pat.row_idx, fp.full.row_idx) and np.array_equal(pat.diag_pos, fp.diag_pos)
    ptr, idx = orc.relaxed_deps(pat)
    level_of, _, _ = orc.levelize(a.n, ptr, idx)
    assert np.array_equal(level_of, glu.levelize(glu.detect_relaxed(fp)).level_of)
