"""The supernodal plan (glu_plan_build_sn) reproduces the reference's
contract-A values bit for bit and is race free (CPU emulation of the
kernel's tasks, tests/sn_emul.py) -- on the reference's own golden cases
and on grids / circuit-like patterns with wide supernodes."""

from __future__ import annotations

import numpy as np
import pytest

import paper_1908_00204_b200 as glu
from paper_1908_00204_b200 import synthetic
from conftest import csc_from_golden, golden_cases, load_golden, pattern_from_golden, random_dd
import sn_emul


def _scatter(fp, a):
    v = np.zeros(fp.nnz)
    rc = glu.numeric._lib.lib.glu_scatter_values(
        fp.n, glu.numeric._lib.ptr(glu.numeric._lib.i64(a.col_ptr)),
        glu.numeric._lib.ptr(glu.numeric._lib.i64(a.row_idx)),
        glu.numeric._lib.ptr(glu.numeric._lib.f64(a.values)),
        glu.numeric._lib.ptr(glu.numeric._lib.i64(fp.full.col_ptr)),
        glu.numeric._lib.ptr(glu.numeric._lib.i64(fp.full.row_idx)), glu.numeric._lib.ptr(v))
    assert rc == -1
    return v


@pytest.mark.parametrize("name", golden_cases())
def test_sn_plan_matches_reference_goldens(name):
    g = load_golden(name)
    a = csc_from_golden(g)
    fp = glu.symbolic_fillin(a.pattern)
    plan = sn_emul.build(fp)
    v, fail = sn_emul.emulate(plan, fp, _scatter(fp, a), float(g["thresh"]))
    if int(g["fail_a"]) >= 0:
        assert fail == int(g["fail_a"])
    else:
        assert fail == -1 and np.array_equal(v, g["lu_a"])


def _oracle_a(fp, a):
    from oracle import oracle as orc

    pat = orc.Pattern.from_fp(fp)
    v, bad = orc.scatter(pat, a.col_ptr, a.row_idx, a.values)
    assert bad == -1
    return v, orc.factor_left_looking(pat, v, 1e-14)


@pytest.mark.parametrize("k,drop,schedule", [(12, 0.0, "all"), (17, 0.1, "all"), (24, 0.0, "all"),
                                             (12, 0.0, "serial"), (17, 0.1, "random"), (20, 0.0, "random")])
def test_sn_plan_grid_bitwise(k, drop, schedule):
    """G3-like grids in nested-dissection order: wide supernodes, panels
    split inside them, relative maps into outside columns.  Every task
    schedule the counters allow gives the reference's bits."""
    a = synthetic.grid5(k, drop=drop, seed=k)
    fp = glu.symbolic_fillin(a.pattern)
    plan = sn_emul.build(fp)
    assert plan["info"]["macs"] == glu.numeric.pattern_flops(fp)[0]
    ref, err = _oracle_a(fp, a)
    assert err == -1
    v, fail = sn_emul.emulate(plan, fp, _scatter(fp, a), schedule=schedule, seed=k)
    assert fail == -1 and np.array_equal(v, ref)


def test_sn_plan_wide_supernode_panels():
    """A dense block (one supernode wider than a panel) below a sparse part."""
    rng = np.random.default_rng(3)
    n = 90
    rows, cols = [], []
    for i in range(n):
        for j in range(n):
            if i == j or (i >= 40 and j >= 40) or rng.uniform() < 0.02:
                rows.append(i)
                cols.append(j)
    vals = rng.uniform(-1, 1, size=len(rows))
    a = glu.to_csc(glu.Triplets(n, n, np.array(rows), np.array(cols), vals))
    rowsum = np.bincount(a.row_idx, weights=np.abs(a.values), minlength=n)
    v = a.values.copy()
    d = a.row_idx == np.repeat(np.arange(n), np.diff(a.col_ptr))
    v[d] = rowsum[a.row_idx[d]] + 1.0
    a = glu.CscMatrix(n, a.col_ptr, a.row_idx, v)
    fp = glu.symbolic_fillin(a.pattern)
    plan = sn_emul.build(fp)
    assert plan["pan"].shape[0] > plan["sn"].shape[0]  # the dense block is split
    ref, err = _oracle_a(fp, a)
    out, fail = sn_emul.emulate(plan, fp, _scatter(fp, a))
    assert err == -1 and fail == -1 and np.array_equal(out, ref)
    out, fail = sn_emul.emulate(plan, fp, _scatter(fp, a), schedule="random", seed=5)
    assert fail == -1 and np.array_equal(out, ref)


@pytest.mark.parametrize("seed,n,dens", [(21, 60, 0.05), (22, 150, 0.02)])
def test_sn_plan_unsymmetric_bitwise(seed, n, dens):
    """Structurally unsymmetric patterns: partial U suffixes inside supernodes."""
    a = random_dd(np.random.default_rng(seed), n, dens)
    fp = glu.symbolic_fillin(a.pattern)
    plan = sn_emul.build(fp)
    ref, err = _oracle_a(fp, a)
    out, fail = sn_emul.emulate(plan, fp, _scatter(fp, a))
    assert err == -1 and fail == -1 and np.array_equal(out, ref)


def test_sn_plan_cfg1_bitwise():
    a = synthetic.make("cfg1")
    fp = glu.symbolic_fillin(a.pattern)
    plan = sn_emul.build(fp)
    assert plan["info"]["macs"] == glu.numeric.pattern_flops(fp)[0]
    ref, err = _oracle_a(fp, a)
    out, fail = sn_emul.emulate(plan, fp, _scatter(fp, a))
    assert err == -1 and fail == -1 and np.array_equal(out, ref)
