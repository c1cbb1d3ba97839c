"""ctypes binding of libglu_b200.so (include/glu_b200.h).

The library is built in-tree by ``__graft_entry__.build()`` (or ``make -C
paper_1908_00204_b200/csrc``).  There is no fallback: if the shared object
is missing the import fails loudly, and every GPU entry point raises if the
CUDA call fails.
"""

from __future__ import annotations

import ctypes
import pathlib

import numpy as np

LIB_PATH = pathlib.Path(__file__).with_name("libglu_b200.so")

GLU_OK = -1
GLU_MISMATCH = -2
GLU_ECUDA = -3
GLU_EINVAL = -4
GLU_ESTRUCT = -5
CONTRACT_A = 0
CONTRACT_B = 1

_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_dbl = ctypes.c_double
_p = ctypes.c_void_p
_pp = ctypes.POINTER(ctypes.c_void_p)
_pi64 = ctypes.POINTER(ctypes.c_int64)
_pi32 = ctypes.POINTER(ctypes.c_int32)

# name -> (restype, argtypes); mirrors include/glu_b200.h
SIGNATURES = {
    "glu_last_error": (_i64, [ctypes.c_char_p, _i64]),
    "glu_version": (ctypes.c_char_p, []),
    "glu_symbolic_fillin": (_i64, [_i64, _p, _p, _i32, _pp, _pi64, _pi64, _pi32]),
    "glu_pattern_nnz": (_i64, [_p]),
    "glu_pattern_export": (None, [_p, _p, _p, _p, _p, _p, _p]),
    "glu_pattern_free": (None, [_p]),
    "glu_csr_view": (_i64, [_i64, _p, _p, _p, _p, _p]),
    "glu_detect_relaxed": (_i64, [_i64, _p, _p, _p, _p, _p, _p, _p]),
    "glu_detect_upward": (_i64, [_i64, _p, _p, _p, _p, _p]),
    "glu_detect_double_u_exact": (_i64, [_i64, _p, _p, _p, _p, _p, _p, _p]),
    "glu_levelize": (_i64, [_i64, _p, _p, _p, _p, _p]),
    "glu_scatter_values": (_i64, [_i64, _p, _p, _p, _p, _p, _p]),
    "glu_find_hazards": (_i64, [_i64, _p, _p, _p, _p, _p, _p, _i64, _p]),
    "glu_plan_build": (_i64, [_i64, _p, _p, _p, _p, _i32, _i64, _i64, _i64, _i32, _pp]),
    "glu_tail_capacity": (_i64, []),
    "glu_host_alloc": (_p, [_i64]),
    "glu_host_free": (None, [_p]),
    "glu_plan_build_sn": (_i64, [_i64, _p, _p, _p, _p, _p, _p, _p, _i32, _pp]),
    "glu_sn_plan_info": (None, [_p, _p]),
    "glu_sn_plan_export": (None, [_p] * 14),
    "glu_schedule_refine": (_i64, [_i64, _p, _p, _p, _p, _p, _p, _i32, _p, _p]),
    "glu_set_fail_levels": (_i64, [_p, _p]),
    "glu_sn_trace": (_i64, [_p, _p, _i64]),
    "glu_plan_info": (None, [_p, _p]),
    "glu_trace_read": (_i64, [_p, _p, _i64]),
    "glu_tail_trace_read": (_i64, [_p, _p, _i64]),
    "glu_kernel_times": (_i64, [_p, _p, _i64]),
    "glu_plan_export": (None, [_p, _p, _p, _p, _p, _p, _p]),
    "glu_plan_free": (None, [_p]),
    "glu_create": (_i64, [_i64, _p, _p, _p, _p, _p, _p, _p, _p, _pp]),
    "glu_destroy": (None, [_p]),
    "glu_set_option": (_i64, [_p, _i64, _i64]),
    "glu_level_times": (_i64, [_p, _p, _i64]),
    "glu_handle_info": (None, [_p, _p]),
    "glu_set_input_pattern": (_i64, [_p, _i64, _p, _p]),
    "glu_scatter_device": (_i64, [_p, _p, _p, _p]),
    "glu_factor_device": (_i64, [_p, _p, _dbl, _p]),
    "glu_factor_device_async": (_i64, [_p, _p, _dbl, _p]),
    "glu_factor_status": (_i64, [_p, _p]),
    "glu_factor_batch_device": (_i64, [_p, _i64, _p, _dbl, _p, _p]),
    "glu_factor_batch_host": (_i64, [_p, _i64, _p, _p, _dbl, _p]),
    "glu_solve_device": (_i64, [_p, _p, _p, _p]),
    "glu_lower_solve_device": (_i64, [_p, _p, _p, _p]),
    "glu_upper_solve_device": (_i64, [_p, _p, _p, _p]),
    "glu_solve_multi_device": (_i64, [_p, _p, _p, _i64, _i64, _i32, _p]),
    "glu_solve_batch_device": (_i64, [_p, _p, _i64, _p, _i64, _i64, _p, _p]),
    "glu_factor_host": (_i64, [_p, _p, _p, _dbl]),
    "glu_solve_host": (_i64, [_p, _p, _p, _p]),
}


class GluError(RuntimeError):
    """A CUDA or argument error inside libglu_b200 (status -3 / -4)."""


def _load():
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
            "(make -C paper_1908_00204_b200/csrc). There is no CPU fallback."
        )
    lib = ctypes.CDLL(str(LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def last_error() -> str:
    buf = ctypes.create_string_buffer(4096)
    lib.glu_last_error(buf, len(buf))
    return buf.value.decode(errors="replace")


def ptr(a: np.ndarray):
    """Raw data pointer of a C-contiguous numpy array."""
    if a is None:
        return None
    assert a.flags.c_contiguous, "array must be C-contiguous"
    return a.ctypes.data_as(ctypes.c_void_p)


def i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def check(rc: int, what: str) -> int:
    """Raise GluError for runtime/argument failures; pass other codes through."""
    if rc in (GLU_ECUDA, GLU_EINVAL):
        raise GluError(f"{what}: {last_error()}")
    return rc
