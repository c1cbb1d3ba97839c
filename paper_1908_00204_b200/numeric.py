"""Numeric factorization, refactorization and solves on the B200
(API of levlu/numeric.py:27-388).

Every factorization and solve below runs in libglu_b200's sm_100a kernels;
there is no CPU fallback.  The per-pattern work (update plan, device upload,
scatter-map build) is cached per (pattern, schedule, contract), so a second
call with the same FilledPattern is a pure refactorization.

Bitwise contracts:
  * contract A -- each entry receives its MACs in ascending source order:
    factor_left_looking, factor_right_looking_seq and
    factor_parallel(deterministic=True) are bit-identical to the reference's.
  * contract B -- level-major order: factor_parallel(deterministic=False) is
    bit-identical to the reference's owner-serialized "atomic" mode.
"""

from __future__ import annotations

import ctypes
import hashlib
import os
import threading
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .depgraph import Hazard, LevelSchedule, detect_relaxed, levelize
from .resource import LevelPlan, ResourceModel, concurrency_cap
from .sparse import CscMatrix
from .symbolic import FilledPattern

DEFAULT_PIVOT_THRESHOLD = 1e-14


class PivotError(ArithmeticError):
    """Zero or near-zero pivot; no numeric pivoting is attempted."""

    def __init__(self, column: int):
        self.column = column
        super().__init__(f"pivot breakdown at column {column}")


class ScheduleHazardError(RuntimeError):
    """A read-write conflict was detected under the given schedule."""

    def __init__(self, hazards):
        self.hazards = hazards
        h = hazards[0]
        super().__init__(
            f"schedule hazard: column {h.writer} writes element {h.element} "
            f"read by column {h.reader} in level {h.level}"
        )


class PatternMismatchError(RuntimeError):
    """A value or update targeted a slot absent from the filled pattern."""


@dataclass(frozen=True)
class FactorOptions:
    zero_pivot_threshold: float = DEFAULT_PIVOT_THRESHOLD
    deterministic: bool = True
    worker_count: int = 1
    resource: ResourceModel | None = None
    detect_races: bool = False

    def __post_init__(self):
        if self.worker_count < 1:
            raise ValueError("worker_count must be >= 1")
        if self.zero_pivot_threshold < 0:
            raise ValueError("zero_pivot_threshold must be non-negative")


@dataclass(frozen=True)
class LuFactors:
    """Unit-lower L and U sharing one value array over the filled pattern."""

    pattern: FilledPattern
    values: np.ndarray

    @property
    def n(self) -> int:
        return self.pattern.n

    def to_scipy(self):
        """(L, U) as scipy CSC matrices, unit diagonal explicit in L."""
        import scipy.sparse as sp

        fp = self.pattern
        cp, rows = fp.full.col_ptr, fp.full.row_idx
        cols = np.repeat(np.arange(fp.n, dtype=np.int64), np.diff(cp))
        low = rows > cols
        eye = sp.identity(fp.n, dtype=self.values.dtype, format="csc")
        L = sp.csc_matrix((self.values[low], (rows[low], cols[low])), shape=(fp.n, fp.n)) + eye
        U = sp.csc_matrix((self.values[~low], (rows[~low], cols[~low])), shape=(fp.n, fp.n))
        return L, U


@dataclass
class FactorStats:
    level_times: list = field(default_factory=list)
    level_modes: list = field(default_factory=list)
    flop_count: int = 0
    peak_concurrent_columns: int = 0


def pattern_flops(fp: FilledPattern) -> tuple[int, int]:
    """(MACs, DIVs) of the pattern: MACs = sum over U entries (i,k) of
    |L(:,i)|, DIVs = nnz(L) (levlu/numeric.py:187-193)."""
    cp = fp.full.col_ptr
    l_len = cp[1:] - fp.diag_pos - 1
    cols = np.repeat(np.arange(fp.n, dtype=np.int64), np.diff(cp))
    upper = fp.full.row_idx < cols
    return int(l_len[fp.full.row_idx[upper]].sum()), int(l_len.sum())


# ---------------------------------------------------------------------------
# device factorizer: pattern + schedule + plan resident on the GPU
# ---------------------------------------------------------------------------
class Factorizer:
    """One (filled pattern, level schedule, contract) resident on the device.

    Owns the libglu_b200 handle: int32 pattern, per-level item/chunk plan and
    the uint16 scatter map (built on the device).  ``factor_host`` is the
    reference-facing path (host buffers in and out); ``factor_device`` works
    in place on device memory (a torch tensor or raw pointer) on a stream.
    """

    def __init__(self, fp: FilledPattern, level_of: np.ndarray, contract: int,
                 max_item_macs: int = 0, threads: int = 0, deep_min: int = 0,
                 tail_max: int | None = None, engine: str = "plan"):
        self.n = fp.n
        self.nnz = fp.nnz
        self.contract = contract
        self.engine = engine
        cp, ri, dp = _lib.i64(fp.full.col_ptr), _lib.i64(fp.full.row_idx), _lib.i64(fp.diag_pos)
        rp, ci, cs = _lib.i64(fp.csr.row_ptr), _lib.i64(fp.csr.col_idx), _lib.i64(fp.csr.csc_pos)
        lv = _lib.i64(level_of)
        plan = ctypes.c_void_p()
        if engine == "sn":
            if contract != _lib.CONTRACT_A:
                raise ValueError("the supernodal engine computes contract A (ascending-source) values")
            rc = _lib.check(_lib.lib.glu_plan_build_sn(self.n, _lib.ptr(cp), _lib.ptr(ri), _lib.ptr(dp),
                                                       _lib.ptr(rp), _lib.ptr(ci), _lib.ptr(cs),
                                                       _lib.ptr(lv), threads, ctypes.byref(plan)),
                            "glu_plan_build_sn")
        elif engine == "plan":
            rc = _lib.check(_lib.lib.glu_plan_build(self.n, _lib.ptr(cp), _lib.ptr(ri), _lib.ptr(dp),
                                                    _lib.ptr(lv), contract, max_item_macs, deep_min,
                                                    _tail_capacity() if tail_max is None else tail_max,
                                                    threads, ctypes.byref(plan)), "glu_plan_build")
        else:
            raise ValueError(f"unknown engine {engine!r} (plan | sn)")
        if rc == _lib.GLU_MISMATCH:
            raise PatternMismatchError("update targeted a structurally absent slot")
        try:
            info = np.zeros(16, dtype=np.int64)
            _lib.lib.glu_plan_info(plan, _lib.ptr(info))
            self.plan_info = dict(zip(("levels", "items", "chunks", "macs", "max_item_macs",
                                       "max_chunks", "deferred_macs", "plan_bytes", "deep_items",
                                       "deep_macs", "epochs", "push_macs", "targets", "tail_t0",
                                       "tail_macs", "reserved"),
                                      info.tolist()))
            if engine == "sn":
                sinfo = np.zeros(16, dtype=np.int64)
                _lib.lib.glu_sn_plan_info(plan, _lib.ptr(sinfo))
                self.sn_info = dict(zip(("supernodes", "panels", "pairs", "map", "pushes", "tasks",
                                         "dblk", "crit_ns", "macs", "plan_bytes", "rg_tasks", "rg_slots",
                                         "rg_macs", "rg_pairs"), sinfo[:14].tolist()))
                self.plan_info.update(macs=self.sn_info["macs"], plan_bytes=self.sn_info["plan_bytes"])
            h = ctypes.c_void_p()
            rc = _lib.check(_lib.lib.glu_create(self.n, _lib.ptr(cp), _lib.ptr(ri), _lib.ptr(dp),
                                                _lib.ptr(rp), _lib.ptr(ci), _lib.ptr(cs),
                                                _lib.ptr(lv), plan, ctypes.byref(h)),
                            "glu_create")
            if rc == _lib.GLU_MISMATCH:
                raise PatternMismatchError("update targeted a structurally absent slot")
        finally:
            _lib.lib.glu_plan_free(plan)
        self._h = h
        self._finalizer = weakref.finalize(self, _lib.lib.glu_destroy, h)
        self._input_key = None
        self._fail_key = _digest(level_of)
        self._lock = threading.Lock()
        if "GLU_POLL_NS" in os.environ:  # tuning: ns between dependency polls (option 6)
            self.set_option(6, int(os.environ["GLU_POLL_NS"]))
        info = np.zeros(12, dtype=np.int64)
        _lib.lib.glu_handle_info(h, _lib.ptr(info))
        self.handle_info = dict(zip(("n", "nnz", "levels", "items", "chunks", "macs",
                                     "device_bytes", "grid", "threads", "lsolve_levels",
                                     "usolve_levels", "sms"), info.tolist()))

    @property
    def handle(self):
        return self._h

    def close(self):
        self._finalizer()

    def set_option(self, key: int, value: int):
        _lib.check(_lib.lib.glu_set_option(self._h, key, value), "glu_set_option")

    def set_fail_levels(self, level_of: np.ndarray):
        """Levels that order pivot failures (factor_parallel reports the
        earliest failing level of the CALLER's schedule, numeric.py:279-285)."""
        key = _digest(level_of)
        if key != self._fail_key:
            _lib.check(_lib.lib.glu_set_fail_levels(self._h, _lib.ptr(_lib.i64(level_of))),
                       "glu_set_fail_levels")
            self._fail_key = key

    def set_input(self, a_col_ptr: np.ndarray, a_row_idx: np.ndarray):
        """Install the A -> A_s slot map (device scatter); cached per A pattern."""
        cp, ri = _lib.i64(a_col_ptr), _lib.i64(a_row_idx)
        last = self._input_key
        if last is not None and _same(last[0], cp) and _same(last[1], ri):
            return  # same A pattern as the installed map (compared, not hashed: cfg4 23 vs 215 ms)
        rc = _lib.check(_lib.lib.glu_set_input_pattern(self._h, len(ri), _lib.ptr(cp), _lib.ptr(ri)),
                        "glu_set_input_pattern")
        if rc >= 0:
            raise PatternMismatchError(f"column {rc} of A has entries outside the filled pattern")
        self._input_key = (cp.copy(), ri.copy())

    def factor_host(self, a_values: np.ndarray, thresh: float) -> tuple[np.ndarray, int]:
        """H2D A values -> device scatter -> factor -> D2H LU values."""
        a = _lib.f64(a_values)
        out = _PINNED.empty(self.nnz) if 8 * self.nnz >= _PINNED_MIN else None
        if out is None:
            out = np.empty(self.nnz, dtype=np.float64)
        rc = _lib.check(_lib.lib.glu_factor_host(self._h, _lib.ptr(a), _lib.ptr(out), float(thresh)),
                        "glu_factor_host")
        return out, rc

    def factor_batch_host(self, a_values: np.ndarray, thresh: float) -> tuple[np.ndarray, np.ndarray]:
        """B value sets (rows, in the input pattern's CSC order) -> (LU values
        [B, nnz], per-set status: -1 or the failing pivot column)."""
        a = np.ascontiguousarray(a_values, dtype=np.float64)
        if a.ndim != 2:
            raise ValueError("a_values must be [batch, nz]")
        out = np.empty((a.shape[0], self.nnz), dtype=np.float64)
        fails = np.empty(a.shape[0], dtype=np.int64)
        _lib.check(_lib.lib.glu_factor_batch_host(self._h, a.shape[0], _lib.ptr(a), _lib.ptr(out),
                                                  float(thresh), _lib.ptr(fails)),
                   "glu_factor_batch_host")
        return out, fails

    def factor_batch_device(self, v, thresh: float, stream=None) -> np.ndarray:
        """In-place factorization of a [B, nnz] device tensor of A_s values;
        returns the per-set status (-1 or the failing pivot column)."""
        batch = int(v.shape[0])
        fails = np.empty(max(batch, 1), dtype=np.int64)
        _lib.check(_lib.lib.glu_factor_batch_device(self._h, batch, _dptr(v), float(thresh),
                                                    _lib.ptr(fails), _stream(stream)),
                   "glu_factor_batch_device")
        return fails[:batch]

    def factor_device(self, v, thresh: float, stream=None) -> int:
        """In-place factorization of device A_s values (torch tensor or int pointer)."""
        return _lib.check(_lib.lib.glu_factor_device(self._h, _dptr(v), float(thresh),
                                                     _stream(stream)), "glu_factor_device")

    def factor_device_async(self, v, thresh: float, stream=None) -> None:
        _lib.check(_lib.lib.glu_factor_device_async(self._h, _dptr(v), float(thresh),
                                                    _stream(stream)), "glu_factor_device_async")

    def status(self, stream=None) -> int:
        return _lib.check(_lib.lib.glu_factor_status(self._h, _stream(stream)), "glu_factor_status")

    def scatter_device(self, a_values, v, stream=None) -> None:
        _lib.check(_lib.lib.glu_scatter_device(self._h, _dptr(a_values), _dptr(v), _stream(stream)),
                   "glu_scatter_device")

    def solve_device(self, lu, x, stream=None) -> int:
        return _lib.check(_lib.lib.glu_solve_device(self._h, _dptr(lu), _dptr(x), _stream(stream)),
                          "glu_solve_device")

    def solve_host(self, lu: np.ndarray, b: np.ndarray, part: str = "both") -> tuple[np.ndarray, int]:
        import torch

        dev = torch.device("cuda", torch.cuda.current_device())
        lu_d = torch.from_numpy(_lib.f64(lu)).to(dev)
        x_d = torch.from_numpy(_lib.f64(b).copy()).to(dev)
        s = torch.cuda.current_stream()
        fn = {"both": _lib.lib.glu_solve_device, "lower": _lib.lib.glu_lower_solve_device,
              "upper": _lib.lib.glu_upper_solve_device}[part]
        rc = _lib.check(fn(self._h, _dptr(lu_d), _dptr(x_d), ctypes.c_void_p(s.cuda_stream)),
                        "glu_solve_device")
        return x_d.cpu().numpy(), rc

    def level_times_s(self) -> list:
        m = int(self.handle_info["levels"])
        ms = np.zeros(max(m, 1), dtype=np.float64)
        k = _lib.lib.glu_level_times(self._h, _lib.ptr(ms), m)
        return (ms[:k] * 1e-3).tolist()


_TAIL_CAP = None


def _tail_capacity() -> int:
    """Dense-tail columns the device's cluster kernel can hold (queried once)."""
    global _TAIL_CAP
    if _TAIL_CAP is None:
        _TAIL_CAP = int(_lib.lib.glu_tail_capacity())
    return _TAIL_CAP


def _dptr(x):
    if x is None:
        return None
    if isinstance(x, int):
        return ctypes.c_void_p(x)
    return ctypes.c_void_p(x.data_ptr())


def _stream(s):
    if s is None:
        import torch

        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(s, int):
        return ctypes.c_void_p(s)
    return ctypes.c_void_p(s.cuda_stream)


def _current_device() -> int:
    import torch

    return torch.cuda.current_device() if torch.cuda.is_available() else -1


_CACHE: dict = {}
# re-entrant: a weakref callback (_drop) can fire from GC while
# get_factorizer holds the lock and allocates
_CACHE_LOCK = threading.RLock()


_DIGESTS: dict = {}
_LIBC = ctypes.CDLL(None)
_LIBC.memcmp.restype = ctypes.c_int
_LIBC.memcmp.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t]


def _same(a: np.ndarray, b: np.ndarray) -> bool:
    """Byte equality of two contiguous arrays of one dtype (memcmp: no
    temporary boolean array; cfg4's A pattern 6 vs 20 ms)."""
    if a.shape != b.shape or a.dtype != b.dtype:
        return False
    if not (a.flags.c_contiguous and b.flags.c_contiguous):
        return bool(np.array_equal(a, b))
    return a.nbytes == 0 or _LIBC.memcmp(a.ctypes.data, b.ctypes.data, a.nbytes) == 0


def _digest(a: np.ndarray) -> bytes:
    """sha1 of an int64 array, remembered per array object: a repeated call
    with the same (unchanged) array costs one comparison instead of a hash
    (cfg4: 3 vs 23 ms per level schedule)."""
    a64 = np.ascontiguousarray(a, dtype=np.int64)
    hit = _DIGESTS.get(id(a))
    if hit is not None and _same(hit[0], a64):
        return hit[1]
    d = hashlib.sha1(a64.tobytes()).digest()
    if len(_DIGESTS) > 16:
        _DIGESTS.clear()
    _DIGESTS[id(a)] = (a64.copy(), d)
    return d


# Per-MAC plans cost ~3.3 B per MAC on the device (and ~2x that on the host
# while building): above this many MACs contract A runs on the supernodal
# engine, whose plan is ~0.17 B per MAC (cfg4: 3.8e10 MACs).  Measured: the
# supernodal engine wins on grids from g400 up (1.2e9 MACs: 7.5 vs ~19 ms)
# and loses on the circuit patterns below the threshold (cfg2 3.0e8 MACs:
# 48 vs 6.8 ms, cfg3: 116 vs 4.9 ms -- few wide supernodes, long chains).
SN_MIN_MACS = int(os.environ.get("GLU_SN_MIN_MACS", 1_000_000_000))
# contract B has no supernodal form: refuse a per-MAC plan beyond this
PLAN_MAX_MACS = int(os.environ.get("GLU_PLAN_MAX_MACS", 12_000_000_000))


def pick_engine(fp: FilledPattern, contract: int) -> str:
    """'sn' (supernodal) or 'plan' (per-MAC items): GLU_ENGINE forces one."""
    forced = os.environ.get("GLU_ENGINE", "auto")
    macs = _flops_cached(fp)[0]
    if contract != _lib.CONTRACT_A:
        if macs > PLAN_MAX_MACS:
            raise _lib.GluError(f"atomic-mode (contract B) factorization needs a per-MAC plan; "
                                f"{macs} MACs exceed GLU_PLAN_MAX_MACS={PLAN_MAX_MACS}")
        return "plan"
    if forced in ("plan", "sn"):
        return forced
    return "sn" if macs >= SN_MIN_MACS else "plan"


def get_factorizer(fp: FilledPattern, level_of: np.ndarray, contract: int,
                   tail: bool = True, engine: str | None = None) -> Factorizer:
    """Cached Factorizer for (fp, schedule, contract, engine); dropped with
    fp.  tail=False builds the batch plan (64-MAC items: the kernel variant
    that loads two value sets per round); either plan keeps the dense
    cluster tail, run as one cluster per value set in batched launches."""
    if engine is None:
        engine = pick_engine(fp, contract)
    if engine == "sn":
        tail = True  # one plan serves single and batched launches
    key = (id(fp), contract, _digest(level_of), tail, engine, _current_device())
    with _CACHE_LOCK:
        hit = _CACHE.get(key)
        if hit is not None and hit[0]() is fp:
            return hit[1]
        # batch plans: 64-MAC items (the kernel variant that
        # loads two value sets per round)
        fz = Factorizer(fp, level_of, contract, tail_max=None,
                        max_item_macs=0 if tail else 64, engine=engine)

        def _drop(_ref, key=key):
            with _CACHE_LOCK:
                ent = _CACHE.pop(key, None)
            if ent is not None:
                ent[1].close()

        _CACHE[key] = (weakref.ref(fp, _drop), fz)
        return fz


_SEQ_LEVELS: dict = {}


def _relaxed_levels(fp: FilledPattern) -> np.ndarray:
    """Relaxed level schedule of fp, cached: the schedule the sequential entry
    points run on (their MAC order is the contract-A order, which is
    schedule independent)."""
    hit = _SEQ_LEVELS.get(id(fp))
    if hit is not None and hit[0]() is fp:
        return hit[1]
    lv = levelize(detect_relaxed(fp)).level_of
    _SEQ_LEVELS[id(fp)] = (weakref.ref(fp, lambda _r, k=id(fp): _SEQ_LEVELS.pop(k, None)), lv)
    return lv


def _value_dtype(values: np.ndarray) -> np.dtype:
    """fp64, or fp32 (the reference's single precision, tests/test_numeric.py:
    203-210): fp32 values are factored and solved in fp64 arithmetic on the
    device and returned rounded to fp32 -- within fp32 rounding of the
    reference's fp32 arithmetic, not bit-identical to it (the bitwise
    contracts are fp64)."""
    dt = np.dtype(values.dtype)
    if dt not in (np.dtype(np.float64), np.dtype(np.float32)):
        raise TypeError(f"the B200 path factors fp64 (or fp32) values; got {dt}")
    return dt


def _require_f64(a: CscMatrix):
    _value_dtype(a.values)


def _check(err: int) -> None:
    if err == _lib.GLU_MISMATCH:
        raise PatternMismatchError("update targeted a structurally absent slot")
    if err >= 0:
        raise PivotError(err)


def plan_levels(fp: FilledPattern, level_of: np.ndarray | None, contract: int) -> np.ndarray:
    """The phase schedule the device plan is built on for a caller's level
    schedule (None: the sequential paths).  Contract A values do not depend
    on the schedule (left-looking order), so it always runs on the relaxed
    schedule; contract B runs on the caller's levels, checked and cut into
    sub-levels where the reference's in-level order matters
    (glu_schedule_refine).  A schedule that puts a source column after its
    target -- the reference would read an unfinished column -- raises
    ScheduleHazardError instead of returning different bits."""
    if level_of is None:
        return _relaxed_levels(fp)
    lv = _lib.i64(level_of)
    key = (id(fp), _digest(lv), contract)
    hit = _PHASES.get(key)
    if hit is not None and hit[0]() is fp:
        return hit[1]
    out = _refine(fp, lv, contract)
    _PHASES[key] = (weakref.ref(fp, lambda _r, k=key: _PHASES.pop(k, None)), out)
    return out


_PHASES: dict = {}


def _refine(fp: FilledPattern, lv: np.ndarray, contract: int) -> np.ndarray:
    if len(lv) != fp.n:
        raise ValueError("level_of must have one entry per column")
    out = np.empty(fp.n, dtype=np.int64)
    bad = np.full(2, -1, dtype=np.int64)
    cp, ri, dp = _lib.i64(fp.full.col_ptr), _lib.i64(fp.full.row_idx), _lib.i64(fp.diag_pos)
    rp, ci = _lib.i64(fp.csr.row_ptr), _lib.i64(fp.csr.col_idx)
    rc = _lib.check(_lib.lib.glu_schedule_refine(fp.n, _lib.ptr(cp), _lib.ptr(ri), _lib.ptr(dp),
                                                 _lib.ptr(rp), _lib.ptr(ci), _lib.ptr(lv), contract,
                                                 _lib.ptr(out), _lib.ptr(bad)), "glu_schedule_refine")
    if rc == _lib.GLU_ESTRUCT:
        i, j = int(bad[0]), int(bad[1])
        raise ScheduleHazardError([Hazard(writer=i, reader=j, element=(i, j), level=int(lv[j]))])
    return _relaxed_levels(fp) if contract == _lib.CONTRACT_A else out


_PINNED_MIN = 32 << 20  # result arrays from this size come from page-locked memory


class _PinnedPool:
    """Page-locked LU result buffers (glu_host_alloc).  glu_factor_host then
    copies final panels into the result by DMA while the kernel runs; into
    fresh pageable memory the copy goes through the driver's staging buffers
    and first-touch page faults (cfg4: ~300 ms for 1.47 GB).  A returned
    array owns its buffer until it and every view of it are gone; the buffer
    then returns to the pool (``keep`` per size) for the next
    refactorization instead of being freed."""

    def __init__(self, keep: int = 2):
        self._free: dict[int, list[int]] = {}
        self._lock = threading.Lock()
        self._keep = keep

    def empty(self, n: int) -> np.ndarray | None:
        nbytes = 8 * n
        with self._lock:
            lst = self._free.get(nbytes)
            addr = lst.pop() if lst else None
        if addr is None:
            addr = _lib.lib.glu_host_alloc(nbytes)
            if not addr:  # no device / pinned memory exhausted: pageable instead
                return None
        buf = (ctypes.c_double * n).from_address(addr)
        weakref.finalize(buf, self._put, addr, nbytes).atexit = False
        return np.frombuffer(buf, dtype=np.float64)

    def _put(self, addr: int, nbytes: int) -> None:
        with self._lock:
            lst = self._free.setdefault(nbytes, [])
            if len(lst) < self._keep:
                lst.append(addr)
                return
        _lib.lib.glu_host_free(addr)


_PINNED = _PinnedPool()


def _factor(a: CscMatrix, fp: FilledPattern, level_of: np.ndarray | None, contract: int,
            thresh: float, by_column: bool, stamps: bool = False) -> tuple[np.ndarray, Factorizer, np.ndarray]:
    _require_f64(a)
    if a.n != fp.n:
        raise PatternMismatchError("matrix and pattern sizes differ")
    phases = plan_levels(fp, level_of, contract)
    fz = get_factorizer(fp, phases, contract)
    dt = _value_dtype(a.values)
    if dt == np.float32:  # the reference's fp32 threshold (numeric.py:268, v.dtype.type)
        thresh = float(np.float32(thresh))
    with fz._lock:
        fz.set_input(a.col_ptr, a.row_idx)
        fz.set_fail_levels(phases if level_of is None or contract != _lib.CONTRACT_A else level_of)
        fz.set_option(2, 1 if by_column else 0)
        fz.set_option(1, 1 if stamps else 0)
        vals, rc = fz.factor_host(np.asarray(a.values, dtype=np.float64), thresh)
    _check(rc)
    return (vals.astype(dt) if dt != np.float64 else vals), fz, phases


def factor_left_looking(a: CscMatrix, fp: FilledPattern,
                        opts: FactorOptions = FactorOptions()) -> LuFactors:
    """Left-looking result (levlu/numeric.py:129-142), computed by the level
    kernel in contract-A order: bitwise the reference's values, failing
    pivot = first failing column."""
    vals, _, _ = _factor(a, fp, None, _lib.CONTRACT_A, opts.zero_pivot_threshold, True)
    return LuFactors(fp, vals)


def factor_right_looking_seq(a: CscMatrix, fp: FilledPattern,
                             opts: FactorOptions = FactorOptions()) -> LuFactors:
    """Sequential right-looking result (levlu/numeric.py:145-159): bitwise
    equal to the left-looking path, so the same contract-A kernel."""
    return factor_left_looking(a, fp, opts)


def find_hazards(fp: FilledPattern, s: LevelSchedule, limit: int = 100000) -> list:
    """Same-level write/read conflicts of the right-looking updates."""
    cp, ri, dp = _lib.i64(fp.full.col_ptr), _lib.i64(fp.full.row_idx), _lib.i64(fp.diag_pos)
    rp, ci = _lib.i64(fp.csr.row_ptr), _lib.i64(fp.csr.col_idx)
    out = np.zeros((limit, 5), dtype=np.int64)
    total = _lib.lib.glu_find_hazards(fp.n, _lib.ptr(cp), _lib.ptr(ri), _lib.ptr(dp), _lib.ptr(rp),
                                      _lib.ptr(ci), _lib.ptr(_lib.i64(s.level_of)), limit,
                                      _lib.ptr(out))
    m = min(int(total), limit)
    return [Hazard(int(w), int(r), (int(i), int(k)), int(l)) for l, w, r, i, k in out[:m]]


def factor_parallel(a: CscMatrix, fp: FilledPattern, schedule: LevelSchedule,
                    plans: list, opts: FactorOptions) -> tuple[LuFactors, FactorStats]:
    """Level-parallel factorization on the B200 (levlu/numeric.py:241-351).

    All levels run in one persistent kernel with a grid barrier per level.
    deterministic=True gives the reference's deterministic (ascending-source)
    values bit for bit, deterministic=False its atomic-mode (level-major)
    values bit for bit; worker_count does not change the result in either
    mode, exactly as in the reference.
    """
    if len(plans) != schedule.level_count:
        raise ValueError("one LevelPlan per level required")
    rm = opts.resource or ResourceModel()
    if opts.detect_races:
        hz = find_hazards(fp, schedule)
        if hz:
            raise ScheduleHazardError(hz)
    contract = _lib.CONTRACT_A if opts.deterministic else _lib.CONTRACT_B
    # per-level GPU completion times (FactorStats.level_times) are opt-in:
    # GLU_LEVEL_TIMES=1 (the stamps cost the per-MAC engine its batched
    # releases); by default level_times holds one 0.0 per level, the length
    # the reference's API guarantees (levlu/numeric.py:321-341)
    stamps = os.environ.get("GLU_LEVEL_TIMES", "0") == "1"
    vals, fz, phases = _factor(a, fp, schedule.level_of, contract, opts.zero_pivot_threshold, False,
                               stamps=stamps)
    caps = [min(concurrency_cap(p, len(c), rm), opts.worker_count, len(c))
            for p, c in zip(plans, schedule.levels)]
    stats = FactorStats(
        level_times=_caller_level_times(fz.level_times_s() if stamps else [], phases,
                                        schedule.level_of, schedule.level_count),
        level_modes=[p.mode.value for p in plans],
        flop_count=sum(_flops_cached(fp)),
        peak_concurrent_columns=max(caps) if caps else 0,
    )
    return LuFactors(fp, vals), stats


def _caller_level_times(phase_s: list, phases: np.ndarray, level_of: np.ndarray, nlev: int) -> list:
    """Per-level GPU times in the caller's schedule from the device's
    per-phase times: a level completes when the last phase holding one of
    its columns completes (the plan may run on refined or relaxed phases)."""
    if not phase_s or len(phases) == 0:
        return [0.0] * nlev
    done = np.cumsum(np.asarray(phase_s, dtype=np.float64))
    ph = np.minimum(np.asarray(phases, dtype=np.int64), len(done) - 1)
    comp = np.zeros(nlev)
    np.maximum.at(comp, np.asarray(level_of, dtype=np.int64), done[ph])
    comp = np.maximum.accumulate(comp)
    return np.diff(np.concatenate([[0.0], comp])).tolist()


_FLOPS: dict = {}


def _flops_cached(fp: FilledPattern) -> tuple[int, int]:
    hit = _FLOPS.get(id(fp))
    if hit is not None and hit[0]() is fp:
        return hit[1]
    f = pattern_flops(fp)
    _FLOPS[id(fp)] = (weakref.ref(fp, lambda _r, k=id(fp): _FLOPS.pop(k, None)), f)
    return f


def refactorize(lu: LuFactors, a_new: CscMatrix, schedule: LevelSchedule | None = None,
                opts: FactorOptions = FactorOptions()) -> LuFactors:
    """New values, same pattern: reuses the device-resident
    pattern, plan and scatter map; only A's values cross the bus."""
    level_of = schedule.level_of if schedule is not None else None
    contract = _lib.CONTRACT_A if opts.deterministic else _lib.CONTRACT_B
    vals, _, _ = _factor(a_new, lu.pattern, level_of, contract, opts.zero_pivot_threshold,
                         schedule is None)
    return LuFactors(lu.pattern, vals)


def refactorize_batch(lu: LuFactors, a_pattern: CscMatrix, values: np.ndarray,
                      schedule: LevelSchedule | None = None,
                      opts: FactorOptions = FactorOptions()) -> tuple[np.ndarray, np.ndarray]:
    """Refactor B value sets on lu's pattern in one call (the cfg5 batch:
    Newton / transient steps).  Row b of `values` holds A's values in
    a_pattern's CSC order (a_pattern.values is ignored).  Returns
    (LU values [B, nnz], status [B]) where status[b] is -1 or the column at
    which set b's pivot broke down (the PivotError the reference would
    raise for that set, numeric.py:27-35)."""
    dt = _value_dtype(a_pattern.values)
    if a_pattern.n != lu.n:
        raise PatternMismatchError("matrix and pattern sizes differ")
    vals = np.ascontiguousarray(values, dtype=np.float64)
    if vals.ndim != 2 or vals.shape[1] != len(a_pattern.row_idx):
        raise ValueError("values must be [batch, nz(A)]")
    contract = _lib.CONTRACT_A if opts.deterministic else _lib.CONTRACT_B
    phases = plan_levels(lu.pattern, schedule.level_of if schedule is not None else None, contract)
    fz = get_factorizer(lu.pattern, phases, contract, tail=False)
    with fz._lock:
        fz.set_input(a_pattern.col_ptr, a_pattern.row_idx)
        fz.set_fail_levels(schedule.level_of if schedule is not None and contract == _lib.CONTRACT_A
                           else phases)
        fz.set_option(2, 1 if schedule is None else 0)
        fz.set_option(1, 0)
        thresh = float(np.float32(opts.zero_pivot_threshold)) if dt == np.float32 else opts.zero_pivot_threshold
        out, fails = fz.factor_batch_host(vals, thresh)
    return (out.astype(dt) if dt != np.float64 else out), fails


def subcolumn_update(fp: FilledPattern, values: np.ndarray, source_j: int, dest_k: int):
    """One rank-1 piece, dest column k -= L(:,j) * U(j,k) (levlu/numeric.py:
    162-184).  A single-pair utility of the reference API, not a path of the
    factorization: evaluated on the host arrays it is given."""
    row_cols = fp.csr.row_cols(source_j)
    t = int(np.searchsorted(row_cols, dest_k))
    if t >= len(row_cols) or row_cols[t] != dest_k:
        raise PatternMismatchError(f"A_s({source_j},{dest_k}) is structurally absent")
    mult = values[fp.csr.row_pos(source_j)[t]]
    dest_rows = fp.full.col_rows(dest_k)
    src = fp.l_positions(source_j)
    r = fp.full.row_idx[src]
    q = np.searchsorted(dest_rows, r)
    ok = (q < len(dest_rows))
    ok[ok] = dest_rows[q[ok]] == r[ok]
    if not ok.all():
        bad = int(r[~ok][0])
        raise PatternMismatchError(f"target slot ({bad},{dest_k}) is structurally absent")
    tgt = fp.full.col_ptr[dest_k] + q
    values[tgt] = values[tgt] - values[src] * mult


def _solve(lu: LuFactors, b: np.ndarray, part: str) -> np.ndarray:
    if len(b) != lu.n:
        raise ValueError("right-hand side length mismatch")
    dt = _value_dtype(lu.values)
    fz = get_factorizer(lu.pattern, _relaxed_levels(lu.pattern), _lib.CONTRACT_A)
    with fz._lock:
        x, rc = fz.solve_host(np.asarray(lu.values, dtype=np.float64),
                              np.asarray(np.asarray(b, dtype=dt), dtype=np.float64), part)
    if rc >= 0:
        raise PivotError(rc)
    return x.astype(dt) if dt != np.float64 else x


def solve_many(lu: LuFactors, b: np.ndarray) -> np.ndarray:
    """Solve A X = B for the columns of B ([n, k]) in one pair of dataflow
    launches; column j of the result is bitwise
    solve(lu, B[:, j])."""
    import torch

    bb = np.asarray(b, dtype=np.float64)
    if bb.ndim != 2 or bb.shape[0] != lu.n:
        raise ValueError("right-hand sides must be [n, k]")
    if lu.values.dtype != np.float64:
        raise TypeError(f"the B200 path solves fp64 factors; got {lu.values.dtype}")
    fz = get_factorizer(lu.pattern, _relaxed_levels(lu.pattern), _lib.CONTRACT_A)
    dev = torch.device("cuda", torch.cuda.current_device())
    with fz._lock:
        lu_d = torch.from_numpy(_lib.f64(lu.values)).to(dev)
        x_d = torch.from_numpy(np.ascontiguousarray(bb.T)).to(dev)  # [k, n]: column j at j * n
        s = torch.cuda.current_stream()
        rc = _lib.check(_lib.lib.glu_solve_multi_device(fz.handle, _dptr(lu_d), _dptr(x_d), bb.shape[1],
                                                        lu.n, 0, ctypes.c_void_p(s.cuda_stream)),
                        "glu_solve_multi_device")
        out = x_d.cpu().numpy().T.copy()
    if rc >= 0:
        raise PivotError(rc)
    return out


def solve_batch(lu: LuFactors, lu_values: np.ndarray, b: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Solve B systems on lu's pattern, each with its own factors -- row b of
    `lu_values` ([B, nnz], e.g. refactorize_batch's output) -- and its own
    right-hand side (row b of `b`, [B, n]), in one pair of dataflow launches
    (the solve after each Newton / transient
    refactorization).  Returns (x [B, n], status [B]): status[b] is -1, or
    the column whose diagonal is exactly zero (the PivotError upper_solve
    raises, levlu/numeric.py:364-373), x[b] then being unspecified.  Every
    solved row is bitwise solve(LuFactors(pattern, lu_values[b]), b[b])."""
    import torch

    vals = np.ascontiguousarray(lu_values, dtype=np.float64)
    bb = np.ascontiguousarray(b, dtype=np.float64)
    if vals.ndim != 2 or vals.shape[1] != lu.pattern.nnz:
        raise ValueError("lu_values must be [batch, nnz]")
    if bb.shape != (vals.shape[0], lu.n):
        raise ValueError("right-hand sides must be [batch, n]")
    nb = vals.shape[0]
    status = np.full(nb, -1, dtype=np.int64)
    if nb == 0:
        return bb.copy(), status
    fz = get_factorizer(lu.pattern, _relaxed_levels(lu.pattern), _lib.CONTRACT_A)
    dev = torch.device("cuda", torch.cuda.current_device())
    with fz._lock:
        lu_d = torch.from_numpy(vals).to(dev)
        x_d = torch.from_numpy(bb.copy()).to(dev)
        s = torch.cuda.current_stream()
        _lib.check(_lib.lib.glu_solve_batch_device(fz.handle, _dptr(lu_d), lu.pattern.nnz, _dptr(x_d), nb,
                                                   lu.n, _lib.ptr(status), ctypes.c_void_p(s.cuda_stream)),
                   "glu_solve_batch_device")
        out = x_d.cpu().numpy()
    return out, status


def lower_solve(lu: LuFactors, b: np.ndarray) -> np.ndarray:
    """L y = b, implicit unit diagonal (levlu/numeric.py:354-361)."""
    return _solve(lu, b, "lower")


def upper_solve(lu: LuFactors, y: np.ndarray) -> np.ndarray:
    """U x = y (levlu/numeric.py:364-373); zero diagonal -> PivotError."""
    return _solve(lu, y, "upper")


def solve(lu: LuFactors, b: np.ndarray) -> np.ndarray:
    """A x = b through both triangular solves (levlu/numeric.py:376-378)."""
    return _solve(lu, b, "both")


def residual(a: CscMatrix, lu: LuFactors) -> float:
    """||A - L U||_F / ||A||_F (verification utility, levlu/numeric.py:381-388)."""
    import scipy.sparse as sp

    L, U = lu.to_scipy()
    A = sp.csc_matrix((a.values, a.row_idx, a.col_ptr), shape=(a.n, a.n))
    diff = (A - L @ U).tocoo()
    num = np.linalg.norm(diff.data)
    den = np.linalg.norm(a.values)
    return float(num / den) if den else float(num)
