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
    lib.orc_int_rows.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                                 _i64p, _i64p]
    lib.orc_total_f64.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _i64p, _f64p]
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


def total(obj, lo: int = 0, hi: int | None = None, lib=None):
    """(contact count, inverse-square sum) over every pair i < j with i in
    [lo, hi) (standard-schedule rows; [0, n) is the whole triangle).  ``lib``
    may be another build of oracle.c (the golden script's -march=native one)."""
    arr = np.ascontiguousarray(np.asarray(obj, dtype=np.float64).reshape(-1, 3))
    hi = len(arr) if hi is None else hi
    c, s = ctypes.c_int64(), ctypes.c_double()
    L = lib or _lib()
    if L.orc_total_f64(arr.ctypes.data, len(arr), lo, hi, ctypes.byref(c), ctypes.byref(s)):
        raise ValueError("bad row range")
    return c.value, s.value


def int_rows(beads, lo: int, hi: int, schedule: str):
    """(exact-coincidence pairs, unit-Manhattan pairs) owned by rows [lo, hi)."""
    arr = np.ascontiguousarray(np.asarray(beads, dtype=np.int64).reshape(-1, 3))
    col, con = ctypes.c_int64(), ctypes.c_int64()
    if _lib().orc_int_rows(arr.ctypes.data, len(arr), 1 if schedule == "balanced" else 0, lo, hi,
                           ctypes.byref(col), ctypes.byref(con)):
        raise ValueError("bad row range")
    return col.value, con.value
