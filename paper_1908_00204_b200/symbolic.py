"""Symbolic fill-in (API of levlu/symbolic.py:21-150), computed natively.

``symbolic_fillin`` calls glu_symbolic_fillin: Gilbert-Peierls reachability
per column (levlu/symbolic.py:66-89) with Eisenstat-Liu symmetric pruning.
The filled pattern is uniquely defined by the input pattern, so the arrays
are identical to the reference's (tests/test_analysis.py).
"""

from __future__ import annotations

import ctypes
import warnings
from dataclasses import dataclass

import numpy as np

from . import _lib
from .sparse import CscPattern, CsrView


class SymbolicError(ValueError):
    """Structurally unusable input: empty column or missing diagonal."""


@dataclass(frozen=True)
class FilledPattern:
    """Fill-in pattern of L+U; column j's U part precedes diag_pos[j], its L
    part follows it (levlu/symbolic.py:25-63)."""

    n: int
    full: CscPattern
    diag_pos: np.ndarray
    csr: CsrView
    nz_before: int

    @property
    def nnz(self) -> int:
        return self.full.nnz

    def u_rows(self, j: int) -> np.ndarray:
        return self.full.row_idx[self.full.col_ptr[j]:self.diag_pos[j]]

    def l_rows(self, j: int) -> np.ndarray:
        return self.full.row_idx[self.diag_pos[j] + 1:self.full.col_ptr[j + 1]]

    def u_positions(self, j: int) -> np.ndarray:
        return np.arange(self.full.col_ptr[j], self.diag_pos[j])

    def l_positions(self, j: int) -> np.ndarray:
        return np.arange(self.diag_pos[j] + 1, self.full.col_ptr[j + 1])

    @property
    def l_col_nonempty(self) -> np.ndarray:
        return (self.full.col_ptr[1:] - self.diag_pos) > 1

    def subcolumns(self, j: int) -> np.ndarray:
        cols = self.csr.row_cols(j)
        return cols[cols > j]


def symbolic_fillin(a: CscPattern, inject_diagonal: bool = True) -> FilledPattern:
    """Exact fill-in pattern; missing diagonals are injected with a warning
    (or raise SymbolicError when ``inject_diagonal`` is false)."""
    n = a.n
    cp, ri = _lib.i64(a.col_ptr), _lib.i64(a.row_idx)
    handle = ctypes.c_void_p()
    injected = ctypes.c_int64()
    bad_col = ctypes.c_int64()
    bad_kind = ctypes.c_int32()
    rc = _lib.lib.glu_symbolic_fillin(n, _lib.ptr(cp), _lib.ptr(ri), int(bool(inject_diagonal)),
                                      ctypes.byref(handle), ctypes.byref(injected),
                                      ctypes.byref(bad_col), ctypes.byref(bad_kind))
    if rc == _lib.GLU_ESTRUCT:
        j = bad_col.value
        if bad_kind.value == 1:
            raise SymbolicError(f"column {j} is structurally empty (singular)")
        raise SymbolicError(f"structural diagonal missing in column {j}")
    _lib.check(rc, "symbolic_fillin")
    try:
        nnz = _lib.lib.glu_pattern_nnz(handle)
        col_ptr = np.empty(n + 1, dtype=np.int64)
        row_idx = np.empty(nnz, dtype=np.int64)
        diag_pos = np.empty(n, dtype=np.int64)
        row_ptr = np.empty(n + 1, dtype=np.int64)
        col_idx = np.empty(nnz, dtype=np.int64)
        csc_pos = np.empty(nnz, dtype=np.int64)
        _lib.lib.glu_pattern_export(handle, _lib.ptr(col_ptr), _lib.ptr(row_idx),
                                    _lib.ptr(diag_pos), _lib.ptr(row_ptr), _lib.ptr(col_idx),
                                    _lib.ptr(csc_pos))
    finally:
        _lib.lib.glu_pattern_free(handle)
    if injected.value:
        k = injected.value
        warnings.warn(f"injected {k} structurally missing diagonal entr{'y' if k == 1 else 'ies'}",
                      stacklevel=2)
    full = CscPattern(n, col_ptr, row_idx)
    return FilledPattern(n, full, diag_pos, CsrView(n, row_ptr, col_idx, csc_pos), int(a.nnz))


def count_fill(fp: FilledPattern) -> tuple[int, int]:
    """(nonzeros before fill, nonzeros after fill)."""
    return fp.nz_before, fp.nnz
