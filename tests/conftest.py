"""Shared test helpers.  `-m gpu` tests need a B200; everything else runs on CPU."""

from __future__ import annotations

import pathlib
import sys

import numpy as np
import pytest

ROOT = pathlib.Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 device (run with -m gpu)")


def golden_cases():
    return sorted(p.stem for p in GOLDEN.glob("*.npz"))


def load_golden(name):
    with np.load(GOLDEN / f"{name}.npz") as d:
        return {k: d[k] for k in d.files}


@pytest.fixture(params=golden_cases())
def golden(request):
    return request.param, load_golden(request.param)


def csc_from_golden(g):
    import paper_1908_00204_b200 as glu

    return glu.CscMatrix(int(g["n"]), g["a_col_ptr"], g["a_row_idx"], g["a_values"])


def pattern_from_golden(g):
    from oracle.oracle import Pattern

    return Pattern(int(g["n"]), g["fp_col_ptr"], g["fp_row_idx"], g["fp_diag_pos"],
                   g["csr_row_ptr"], g["csr_col_idx"], g["csr_csc_pos"])


def random_dd(rng, n, density):
    """Random diagonally dominant matrix with a full diagonal."""
    import paper_1908_00204_b200 as glu

    m = max(int(density * n * n), n)
    rows = np.concatenate([rng.integers(0, n, size=m), np.arange(n)])
    cols = np.concatenate([rng.integers(0, n, size=m), np.arange(n)])
    vals = np.concatenate([rng.uniform(-1.0, 1.0, size=m), np.zeros(n)])
    a = glu.to_csc(glu.Triplets(n, n, rows, cols, vals))
    rowsum = np.bincount(a.row_idx, weights=np.abs(a.values), minlength=n)
    v = a.values.copy()
    cols_of = np.repeat(np.arange(n), np.diff(a.col_ptr))
    d = a.row_idx == cols_of
    v[d] = rowsum[a.row_idx[d]] + 1.0
    return glu.CscMatrix(a.n, a.col_ptr, a.row_idx, v)


def has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False
