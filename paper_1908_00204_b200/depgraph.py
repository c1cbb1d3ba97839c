"""Column dependencies and levelization (API of levlu/depgraph.py).

The detectors (upward, relaxed = paper Alg. 4, the exact GLU2.0 double-U
rule; levlu/depgraph.py:96-156), ``levelize`` (:159-170) and
``simulate_hazards`` (:173-205) run natively on the host and keep edge
lists in CSR form; ``DependencyGraph.deps`` materializes the reference's
list-of-arrays view on demand, and ``DependencyGraph(n, deps, method)``
builds a graph from that view as the reference's dataclass does.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .symbolic import FilledPattern


class DetectMethod(enum.Enum):
    UPWARD = "upward"
    DOUBLE_U_EXACT = "exact"
    RELAXED = "relaxed"


class DependencyGraph:
    """Per-column sorted lists of strictly smaller columns each column needs
    (levlu/depgraph.py:27-38: DependencyGraph(n, deps, method))."""

    def __init__(self, n: int, deps: list, method: DetectMethod):
        self.n = n
        self.method = method
        self._deps = list(deps)
        if len(self._deps) != n:
            raise ValueError("one dependency list per column")
        lens = np.array([len(d) for d in self._deps], dtype=np.int64)
        self.dep_ptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        self.dep_idx = (np.concatenate([np.asarray(d, dtype=np.int64) for d in self._deps])
                        if self.dep_ptr[-1] else np.empty(0, dtype=np.int64))

    @classmethod
    def from_csr(cls, n: int, dep_ptr: np.ndarray, dep_idx: np.ndarray, method: DetectMethod):
        g = cls.__new__(cls)
        g.n, g.method, g.dep_ptr, g.dep_idx, g._deps = n, method, dep_ptr, dep_idx, None
        return g

    @property
    def deps(self) -> list:
        if self._deps is None:
            p, d = self.dep_ptr, self.dep_idx
            self._deps = [d[p[j]:p[j + 1]] for j in range(self.n)]
        return self._deps

    def __eq__(self, other):
        if not isinstance(other, DependencyGraph):
            return NotImplemented
        return (self.n == other.n and self.method == other.method and
                np.array_equal(self.dep_ptr, other.dep_ptr) and np.array_equal(self.dep_idx, other.dep_idx))

    __hash__ = None

    @property
    def edge_count(self) -> int:
        return int(self.dep_ptr[-1]) if self.n else 0

    def edge_set(self) -> set:
        cols = np.repeat(np.arange(self.n, dtype=np.int64), np.diff(self.dep_ptr))
        return set(zip(cols.tolist(), self.dep_idx.tolist()))


@dataclass(frozen=True)
class LevelSchedule:
    """Ordered levels of mutually independent columns."""

    levels: list
    level_of: np.ndarray

    @property
    def level_count(self) -> int:
        return len(self.levels)


@dataclass(frozen=True)
class Hazard:
    writer: int
    reader: int
    element: tuple  # (i, k) position in the filled pattern
    level: int


@dataclass(frozen=True)
class HazardReport:
    hazards: list

    def __len__(self) -> int:
        return len(self.hazards)


@dataclass
class LevelStats:
    """Per-level size and max subcolumn count; modes filled by plan_schedule."""

    sizes: list
    max_subcolumns: list
    modes: list = field(default_factory=list)

    @property
    def level_count(self) -> int:
        return len(self.sizes)


def _fp_arrays(fp: FilledPattern):
    return (_lib.i64(fp.full.col_ptr), _lib.i64(fp.full.row_idx), _lib.i64(fp.diag_pos),
            _lib.i64(fp.csr.row_ptr), _lib.i64(fp.csr.col_idx))


def detect_relaxed(fp: FilledPattern) -> DependencyGraph:
    """Upward edges plus one left scan of each L row (superset of exact)."""
    cp, ri, dp, rp, ci = _fp_arrays(fp)
    n = fp.n
    dep_ptr = np.zeros(n + 1, dtype=np.int64)
    dep_idx = np.empty(max(int(cp[-1]) if n else 0, 1), dtype=np.int64)
    e = _lib.check(_lib.lib.glu_detect_relaxed(n, _lib.ptr(cp), _lib.ptr(ri), _lib.ptr(dp),
                                               _lib.ptr(rp), _lib.ptr(ci), _lib.ptr(dep_ptr),
                                               _lib.ptr(dep_idx)), "detect_relaxed")
    return DependencyGraph.from_csr(n, dep_ptr, dep_idx[:e].copy(), DetectMethod.RELAXED)


def detect_upward(fp: FilledPattern) -> DependencyGraph:
    """U-pattern rule only (unsafe for parallel right-looking updates)."""
    cp, ri, dp, _, _ = _fp_arrays(fp)
    n = fp.n
    dep_ptr = np.zeros(n + 1, dtype=np.int64)
    dep_idx = np.empty(max(int(cp[-1]) if n else 0, 1), dtype=np.int64)
    e = _lib.check(_lib.lib.glu_detect_upward(n, _lib.ptr(cp), _lib.ptr(ri), _lib.ptr(dp),
                                              _lib.ptr(dep_ptr), _lib.ptr(dep_idx)),
                   "detect_upward")
    return DependencyGraph.from_csr(n, dep_ptr, dep_idx[:e].copy(), DetectMethod.UPWARD)


def detect_double_u_exact(fp: FilledPattern) -> DependencyGraph:
    """Exact GLU2.0 detection (levlu/depgraph.py:129-156): upward edges plus
    the double-U rule -- t depends on i (L(t,i) != 0) when a row j in
    {t} u L(:,t) shares a column k > t with row i."""
    cp, ri, dp, rp, ci = _fp_arrays(fp)
    n = fp.n
    dep_ptr = np.zeros(n + 1, dtype=np.int64)
    dep_idx = np.empty(max(int(cp[-1]) if n else 0, 1), dtype=np.int64)
    e = _lib.check(_lib.lib.glu_detect_double_u_exact(n, _lib.ptr(cp), _lib.ptr(ri), _lib.ptr(dp),
                                                      _lib.ptr(rp), _lib.ptr(ci), _lib.ptr(dep_ptr),
                                                      _lib.ptr(dep_idx)), "detect_double_u_exact")
    return DependencyGraph.from_csr(n, dep_ptr, dep_idx[:e].copy(), DetectMethod.DOUBLE_U_EXACT)


def simulate_hazards(fp: FilledPattern, s: LevelSchedule) -> HazardReport:
    """Same-level (writer, reader) pairs whose right-looking write set meets
    the reader's multiplier read set (levlu/depgraph.py:173-205), in the
    reference's order: level, writer, reader, element.  Evaluated natively
    in O(MACs) instead of the reference's per-level set products."""
    seen = np.concatenate(s.levels) if s.levels else np.empty(0, dtype=np.int64)
    if len(seen) != fp.n or len(np.unique(seen)) != fp.n:
        raise ValueError("schedule is not a partition of the columns")
    cp, ri, dp, rp, ci = _fp_arrays(fp)
    lv = _lib.i64(s.level_of)
    cap = 1 << 16
    while True:
        out = np.zeros((cap, 5), dtype=np.int64)
        total = int(_lib.lib.glu_find_hazards(fp.n, _lib.ptr(cp), _lib.ptr(ri), _lib.ptr(dp), _lib.ptr(rp),
                                              _lib.ptr(ci), _lib.ptr(lv), cap, _lib.ptr(out)))
        if total <= cap:
            break
        cap = 4 * total
    return HazardReport([Hazard(int(w), int(r), (int(i), int(k)), int(l)) for l, w, r, i, k in out[:total]])


def _graph_csr(g) -> tuple[np.ndarray, np.ndarray]:
    if isinstance(g, DependencyGraph):
        return _lib.i64(g.dep_ptr), _lib.i64(g.dep_idx)
    # a reference levlu.DependencyGraph (list of arrays)
    lens = np.array([len(d) for d in g.deps], dtype=np.int64)
    ptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    idx = np.concatenate(g.deps).astype(np.int64) if ptr[-1] else np.empty(0, np.int64)
    return ptr, _lib.i64(idx)


def levelize(g) -> LevelSchedule:
    """level(j) = 1 + max level of its dependencies; ascending columns per level."""
    n = g.n
    ptr, idx = _graph_csr(g)
    level_of = np.zeros(n, dtype=np.int64)
    level_ptr = np.zeros(n + 1, dtype=np.int64)
    level_cols = np.empty(max(n, 1), dtype=np.int64)
    nl = _lib.check(_lib.lib.glu_levelize(n, _lib.ptr(ptr), _lib.ptr(idx if len(idx) else
                                                                      np.zeros(1, np.int64)),
                                          _lib.ptr(level_of), _lib.ptr(level_ptr),
                                          _lib.ptr(level_cols)), "levelize")
    levels = [level_cols[level_ptr[i]:level_ptr[i + 1]] for i in range(nl)]
    return LevelSchedule(levels, level_of)


def subcolumn_counts(fp: FilledPattern) -> np.ndarray:
    """Per row j, the number of entries right of the diagonal (|subcolumns(j)|)."""
    rp, ci = fp.csr.row_ptr, fp.csr.col_idx
    rows = np.repeat(np.arange(fp.n, dtype=np.int64), np.diff(rp))
    return np.bincount(rows[ci > rows], minlength=fp.n).astype(np.int64)


def level_stats(fp: FilledPattern, s: LevelSchedule) -> LevelStats:
    """Per-level size and maximum subcolumn count (levlu/depgraph.py:208-215)."""
    sub = subcolumn_counts(fp)
    sizes = [len(c) for c in s.levels]
    max_subs = [int(sub[c].max()) if len(c) else 0 for c in s.levels]
    return LevelStats(sizes, max_subs)
