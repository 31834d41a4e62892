"""ctypes wrapper of oracle/liboracle.so -- TEST INFRASTRUCTURE ONLY."""

from __future__ import annotations

import ctypes
from functools import lru_cache

import numpy as np

from .build import build

_i64p = ctypes.POINTER(ctypes.c_int64)
_f64p = ctypes.POINTER(ctypes.c_double)


@lru_cache(maxsize=1)
def _lib():
    lib = ctypes.CDLL(str(build()))
    lib.orc_rows_f64.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int64,
                                 ctypes.c_int64, _i64p, _f64p, _i64p]
    lib.orc_int_pairs.argtypes = [ctypes.c_void_p, ctypes.c_int64, _i64p, _i64p]
    return lib


def rows(obj, lo: int, hi: int, schedule: str):
    """(contact count, inverse-square sum, pairs) owned by rows [lo, hi)."""
    arr = np.ascontiguousarray(np.asarray(obj, dtype=np.float64).reshape(-1, 3))
    c, p = ctypes.c_int64(), ctypes.c_int64()
    s = ctypes.c_double()
    rc = _lib().orc_rows_f64(arr.ctypes.data, len(arr), 1 if schedule == "balanced" else 0, lo, hi,
                             ctypes.byref(c), ctypes.byref(s), ctypes.byref(p))
    if rc:
        raise ValueError("bad row range")
    return c.value, s.value, p.value


def int_pairs(beads):
    """(exact-coincidence pairs, unit-Manhattan pairs) over all i < j."""
    arr = np.ascontiguousarray(np.asarray(beads, dtype=np.int64).reshape(-1, 3))
    col, con = ctypes.c_int64(), ctypes.c_int64()
    _lib().orc_int_pairs(arr.ctypes.data, len(arr), ctypes.byref(col), ctypes.byref(con))
    return col.value, con.value
