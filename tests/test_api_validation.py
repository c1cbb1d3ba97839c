"""Argument validation of the batch / multi-RHS entry points: rejected on the
host, before any device work (runs without a GPU)."""

import numpy as np
import pytest

import paper_1908_00204_b200 as glu
from conftest import csc_from_golden, load_golden


@pytest.fixture
def lu5():
    g = load_golden("diag5")
    fp = glu.symbolic_fillin(csc_from_golden(g).pattern)
    return glu.LuFactors(fp, np.asarray(g["lu_a"], dtype=np.float64))


def test_solve_many_rejects_bad_shapes(lu5):
    with pytest.raises(ValueError):
        glu.solve_many(lu5, np.ones(5))          # not [n, k]
    with pytest.raises(ValueError):
        glu.solve_many(lu5, np.ones((4, 2)))     # wrong n


def test_solve_batch_rejects_bad_shapes(lu5):
    vals = np.tile(lu5.values, (3, 1))
    with pytest.raises(ValueError):
        glu.solve_batch(lu5, vals[:, :-1], np.ones((3, 5)))   # not [B, nnz]
    with pytest.raises(ValueError):
        glu.solve_batch(lu5, vals, np.ones((2, 5)))           # B mismatch
    with pytest.raises(ValueError):
        glu.solve_batch(lu5, vals, np.ones((3, 4)))           # n mismatch
    x, st = glu.solve_batch(lu5, vals[:0], np.ones((0, 5)))   # empty batch: no device work
    assert x.shape == (0, 5) and st.shape == (0,)


def test_refactorize_batch_rejects_bad_shapes(lu5):
    g = load_golden("diag5")
    a = csc_from_golden(g)
    with pytest.raises(ValueError):
        glu.refactorize_batch(lu5, a, np.ones((2, len(a.row_idx) + 1)))
    with pytest.raises(TypeError):  # fp64 / fp32 only
        glu.refactorize_batch(lu5, glu.CscMatrix(a.n, a.col_ptr, a.row_idx,
                                                 a.values.astype(np.complex128)), np.ones((2, 5)))
