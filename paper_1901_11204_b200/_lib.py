"""ctypes binding of libpaircount.so (include/paircount.h).

This is the only place the package touches native code.  There is no CPU
fallback: if the shared library is missing, or no CUDA device is visible,
every compute entry point raises ``PaircountUnavailable`` (a RuntimeError).
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("PAIRCOUNT_LIB", str(HERE / "libpaircount.so")))

# --- codes (include/paircount.h) -------------------------------------------
PC_OK = 0
PC_ERR_CUDA = -1
PC_ERR_ARG = 1
PC_ERR_DOMAIN = 2
PC_ERR_RANGE = 3
PC_ERR_OVERFLOW = 4
PC_ERR_ODD = 5

PC_F32, PC_F64, PC_I32, PC_I64 = 0, 1, 2, 3
PC_STANDARD, PC_BALANCED = 0, 1
PC_COLLISION, PC_COLLISION_INVSQ, PC_COINCIDE, PC_MANHATTAN1 = 1, 2, 3, 4
PC_TILE_AUTO, PC_TILE_PER_ROW_TILE, PC_TILE_FLAT, PC_TILE_TC, PC_TILE_SORTED, PC_TILE_KEY = 0, 1, 2, 3, 4, 5
PC_TILE_THREAD_ROW = 6

SCHEDULE_CODES = {"standard": PC_STANDARD, "balanced": PC_BALANCED}
DTYPE_CODES = {np.dtype(np.float32): PC_F32, np.dtype(np.float64): PC_F64,
               np.dtype(np.int32): PC_I32, np.dtype(np.int64): PC_I64}

# Every symbol include/paircount.h declares (checked by tests/test_abi.py).
EXPORTED = (
    "pc_last_error", "pc_version", "pc_device_count", "pc_set_device", "pc_device_alloc",
    "pc_device_free", "pc_memcpy_h2d", "pc_memcpy_d2h", "pc_stream_sync",
    "pc_pairs_workspace_bytes", "pc_pairs", "pc_pairs_async", "pc_pairs_host", "pc_pairs_multi", "pc_pairs_batch",
    "pc_pairs_part_async", "pc_pairs_part_host", "pc_pairs_last_profile", "pc_pairs_profile_read",
    "pc_last_launch_count", "pc_kernel_timing", "pc_kernel_timing_read", "pc_kernel_timing_read_split", "pc_lattice_grid_cells", "pc_lattice_key_bytes",
    "pc_lattice_collisions", "pc_lattice_contacts", "pc_lattice_reset_keys", "pc_lattice_clear",
    "pc_lattice_collisions_batch", "pc_lattice_collisions_vectors", "pc_lattice_collisions_multi",
    "pc_lattice_reset_beads", "pc_grid_count_nonzero", "pc_microbench",
)


class PaircountUnavailable(RuntimeError):
    """libpaircount.so is not built or no CUDA device is visible."""


class PaircountError(RuntimeError):
    """A CUDA call inside libpaircount failed."""


class PairsResult(ctypes.Structure):
    _fields_ = [("count", ctypes.c_int64), ("sum", ctypes.c_double), ("pairs", ctypes.c_int64),
                ("exact_checks", ctypes.c_int64), ("error", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class PairsProfile(ctypes.Structure):
    """pc_pairs_profile: what the kernels of one call did (include/paircount.h)."""
    _fields_ = [("chunks_gram", ctypes.c_int64), ("chunks_main", ctypes.c_int64), ("chunks_near", ctypes.c_int64),
                ("chunks_far", ctypes.c_int64), ("chunks_edge", ctypes.c_int64), ("rows_rescanned", ctypes.c_int64),
                ("exact_checks", ctypes.c_int64), ("claims", ctypes.c_int64), ("pairs", ctypes.c_int64),
                ("pairs_per_chunk", ctypes.c_int64), ("kernel", ctypes.c_int32), ("f64_taken", ctypes.c_int32),
                ("chunks_tc", ctypes.c_int64)]

    def as_dict(self) -> dict:
        return {name: int(getattr(self, name)) for name, _ in self._fields_}


class LatticeResult(ctypes.Structure):
    _fields_ = [("count", ctypes.c_int64), ("beads_processed", ctypes.c_int64),
                ("cells_touched", ctypes.c_int64), ("doubled", ctypes.c_int64),
                ("error", ctypes.c_int32), ("reserved", ctypes.c_int32), ("detail", ctypes.c_int64)]


_vp, _i32, _i64, _sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
_SIGS = {
    "pc_last_error": ([], ctypes.c_char_p),
    "pc_version": ([], ctypes.c_char_p),
    "pc_device_count": ([ctypes.POINTER(_i32)], ctypes.c_int),
    "pc_set_device": ([_i32], ctypes.c_int),
    "pc_device_alloc": ([_sz, ctypes.POINTER(_vp)], ctypes.c_int),
    "pc_device_free": ([_vp], ctypes.c_int),
    "pc_memcpy_h2d": ([_vp, _vp, _sz, _vp], ctypes.c_int),
    "pc_memcpy_d2h": ([_vp, _vp, _sz, _vp], ctypes.c_int),
    "pc_stream_sync": ([_vp], ctypes.c_int),
    "pc_pairs_workspace_bytes": ([_i64, _i32], _sz),
    "pc_pairs": ([_vp, _i32, _i64, _i32, _i32, _i32, _i32, _vp, _vp, _sz, _vp, _vp], ctypes.c_int),
    "pc_pairs_async": ([_vp, _i32, _i64, _i32, _i32, _i32, _i32, _vp, _vp, _sz, _vp, _vp], ctypes.c_int),
    "pc_pairs_host": ([_vp, _i32, _i64, _i32, _i32, _i32, _i32, _vp, _vp], ctypes.c_int),
    "pc_pairs_multi": ([_vp, _i32, _i64, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp], ctypes.c_int),
    "pc_pairs_part_async": ([_vp, _i32, _i64, _i32, _i32, _i32, _i64, _i64, _i32, _i32, _vp, _sz, _vp, _vp],
                            ctypes.c_int),
    "pc_pairs_part_host": ([_vp, _i32, _i64, _i32, _i32, _i32, _i64, _i64, _i32, _i32, _vp], ctypes.c_int),
    "pc_pairs_last_profile": ([_vp], ctypes.c_int),
    "pc_pairs_profile_read": ([_vp, _i64, _vp, _vp], ctypes.c_int),
    "pc_pairs_batch": ([_vp, _vp, _i32, _i32, _i32, _vp, _vp], ctypes.c_int),
    "pc_last_launch_count": ([], _i32),
    "pc_kernel_timing": ([_i32], ctypes.c_int),
    "pc_kernel_timing_read": ([ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_i32)], ctypes.c_int),
    "pc_kernel_timing_read_split": ([ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_i32)], ctypes.c_int),
    "pc_lattice_grid_cells": ([_i64], _i64),
    "pc_lattice_key_bytes": ([_i64], _i32),
    "pc_lattice_collisions": ([_vp, _i32, _i32, _i64, _i64, _vp, _vp, _i32, _vp, _vp], ctypes.c_int),
    "pc_lattice_contacts": ([_vp, _i32, _i32, _i64, _i64, _vp, _vp, _i32, _vp, _vp], ctypes.c_int),
    "pc_lattice_reset_keys": ([_vp, _i64, _vp, _i64, _vp], ctypes.c_int),
    "pc_lattice_reset_beads": ([_vp, _i32, _i32, _i64, _i64, _vp, _vp, _vp], ctypes.c_int),
    "pc_lattice_clear": ([_vp, _i64, _vp], ctypes.c_int),
    "pc_lattice_collisions_batch": ([_vp, _i32, _i32, _vp, _i32, _i64, _vp, _vp], ctypes.c_int),
    "pc_lattice_collisions_vectors": ([_vp, _vp, _i32, _i32, _i64, _vp, _vp], ctypes.c_int),
    "pc_lattice_collisions_multi": ([_vp, _i32, _i64, _i64, _i32, _vp, _vp, _vp], ctypes.c_int),
    "pc_grid_count_nonzero": ([_vp, _i64, ctypes.POINTER(_i64), _vp], ctypes.c_int),
    "pc_microbench": ([_i32, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)], ctypes.c_int),
}

_lock = threading.Lock()
_handle = None
_device_checked = False
_tls = threading.local()  # the CUDA current device is per host thread: set it in each calling thread


def load(require_device: bool = True):
    """Load (once) and return the ctypes handle; fail loudly if unavailable."""
    global _handle, _device_checked
    with _lock:
        if _handle is None:
            if not LIB_PATH.exists():
                raise PaircountUnavailable(
                    f"{LIB_PATH} is not built; run `python -m paper_1901_11204_b200.build` "
                    "(there is no CPU fallback)")
            lib = ctypes.CDLL(str(LIB_PATH))
            for name, (args, res) in _SIGS.items():
                fn = getattr(lib, name, None)
                if fn is None:  # an older build under PAIRCOUNT_LIB (A/B timing); test_abi checks the shipped one
                    continue
                fn.argtypes = args
                fn.restype = res
            _handle = lib
        if require_device and not _device_checked:
            cnt = ctypes.c_int32(0)
            rc = _handle.pc_device_count(ctypes.byref(cnt))
            if rc != PC_OK or cnt.value < 1:
                raise PaircountUnavailable(
                    "no CUDA device visible to libpaircount (there is no CPU fallback): "
                    + _handle.pc_last_error().decode())
            _device_checked = True
        if require_device and not getattr(_tls, "device_set", False):
            # PAIRCOUNT_DEVICE pins the device; without it the thread's current CUDA
            # device (e.g. torch.cuda.set_device) is left alone
            if "PAIRCOUNT_DEVICE" in os.environ:
                check(_handle.pc_set_device(int(os.environ["PAIRCOUNT_DEVICE"])))
            _tls.device_set = True
        return _handle


def last_error() -> str:
    return load(require_device=False).pc_last_error().decode()


def check(rc: int) -> None:
    if rc == PC_ERR_CUDA:
        raise PaircountError(last_error())
    if rc == PC_ERR_ARG:
        raise ValueError(last_error())


def device_count() -> int:
    """CUDA devices visible to libpaircount (0 when none)."""
    cnt = ctypes.c_int32(0)
    if load(require_device=False).pc_device_count(ctypes.byref(cnt)) != PC_OK:
        return 0
    return int(cnt.value)


def launches() -> int:
    """Kernel launches issued by the last pairs/lattice call on this thread."""
    return int(load(require_device=False).pc_last_launch_count())


# --- all-pairs --------------------------------------------------------------

def pairs_host(xyz: np.ndarray, interaction: int, schedule: int, bounds, tiling: int = PC_TILE_AUTO):
    """Run pc_pairs_host on a C-contiguous (n, 3) array; returns PairsResult[]."""
    lib = load()
    arr = np.ascontiguousarray(xyz)
    code = DTYPE_CODES[arr.dtype]
    b = np.ascontiguousarray(np.asarray(bounds, dtype=np.int64))
    nr = len(b) - 1
    res = (PairsResult * nr)()
    rc = lib.pc_pairs_host(arr.ctypes.data, code, len(arr), interaction, schedule, tiling, nr,
                           b.ctypes.data, ctypes.addressof(res))
    check(rc)
    return list(res)


def pairs_part_host(xyz: np.ndarray, interaction: int, schedule: int, lo: int, hi: int, part: int, nparts: int,
                    tiling: int = PC_TILE_AUTO):
    """pc_pairs_part_host: row tiles part, part + nparts, ... of [lo, hi); returns one PairsResult."""
    lib = load()
    arr = np.ascontiguousarray(xyz)
    res = PairsResult()
    check(lib.pc_pairs_part_host(arr.ctypes.data, DTYPE_CODES[arr.dtype], len(arr), interaction, schedule, tiling,
                                 lo, hi, part, nparts, ctypes.byref(res)))
    return res


def pairs_part_async(xyz_ptr: int, dtype_code: int, n: int, interaction: int, schedule: int, lo: int, hi: int,
                     part: int, nparts: int, workspace_ptr: int, workspace_bytes: int, results_dev_ptr: int,
                     stream_ptr: int, tiling: int = PC_TILE_AUTO) -> None:
    """Device-pointer entry of pc_pairs_part_async: enqueue, no synchronisation."""
    check(load().pc_pairs_part_async(xyz_ptr, dtype_code, n, interaction, schedule, tiling, lo, hi, part, nparts,
                                     workspace_ptr, workspace_bytes, results_dev_ptr, stream_ptr))


def last_profile() -> PairsProfile:
    """Profile of the last pc_pairs_host / pc_pairs_part_host call on this thread."""
    prof = PairsProfile()
    check(load().pc_pairs_last_profile(ctypes.byref(prof)))
    return prof


def profile_read(workspace_ptr: int, n: int, stream_ptr: int) -> PairsProfile:
    """Profile of the last device-pointer call on this workspace (synchronises the stream)."""
    prof = PairsProfile()
    check(load().pc_pairs_profile_read(workspace_ptr, n, ctypes.byref(prof), stream_ptr))
    return prof


def pairs_multi(xyz: np.ndarray, interaction: int, schedule: int, devices, bounds, tiling: int = PC_TILE_AUTO):
    """pc_pairs_multi: slab d of the rows on devices[d]; returns (per-device results, total)."""
    lib = load()
    arr = np.ascontiguousarray(xyz)
    devs = np.ascontiguousarray(np.asarray(devices, dtype=np.int32))
    b = np.ascontiguousarray(np.asarray(bounds, dtype=np.int64))
    if len(b) != len(devs) + 1:
        raise ValueError("need len(devices) + 1 slab bounds")
    per = (PairsResult * len(devs))()
    tot = PairsResult()
    check(lib.pc_pairs_multi(arr.ctypes.data, DTYPE_CODES[arr.dtype], len(arr), interaction, schedule, tiling,
                             len(devs), devs.ctypes.data, b.ctypes.data, ctypes.addressof(per), ctypes.byref(tot)))
    return list(per), tot


def host_address(arr: np.ndarray) -> int:
    """Data pointer of a C-contiguous array (the buffer-protocol route is ~3x
    cheaper than ``arr.ctypes.data``, which matters at 1000 vectors a call)."""
    try:
        return ctypes.addressof(ctypes.c_char.from_buffer(arr))
    except (TypeError, ValueError):  # read-only or empty buffer
        return arr.ctypes.data


def pairs_batch(arrays, interaction: int):
    """pc_pairs_batch over a list of C-contiguous (n, 3) arrays of one dtype; returns PairsResult[]."""
    lib = load()
    if not arrays:
        return []
    dt = arrays[0].dtype
    if any(a.dtype != dt for a in arrays):
        raise ValueError("pairs_batch needs one dtype for all vectors")
    ptrs = np.array([host_address(a) for a in arrays], dtype=np.uintp)
    lengths = np.array([len(a) for a in arrays], dtype=np.int64)
    res = (PairsResult * len(arrays))()
    check(lib.pc_pairs_batch(ptrs.ctypes.data, lengths.ctypes.data, DTYPE_CODES[dt], len(arrays), interaction,
                             ctypes.addressof(res), None))
    return list(res)


def pairs_async(xyz_ptr: int, dtype_code: int, n: int, interaction: int, schedule: int, bounds_host: np.ndarray,
                workspace_ptr: int, workspace_bytes: int, results_dev_ptr: int, stream_ptr: int,
                tiling: int = PC_TILE_AUTO) -> None:
    """Device-pointer entry (bench / torch users): enqueue, no synchronisation."""
    lib = load()
    b = np.ascontiguousarray(bounds_host, dtype=np.int64)
    rc = lib.pc_pairs_async(xyz_ptr, dtype_code, n, interaction, schedule, tiling, len(b) - 1, b.ctypes.data,
                            workspace_ptr, workspace_bytes, results_dev_ptr, stream_ptr)
    check(rc)


def workspace_bytes(n: int, nranges: int = 1) -> int:
    return int(load(require_device=False).pc_pairs_workspace_bytes(n, nranges))


def kernel_timing(enable: bool) -> None:
    check(load().pc_kernel_timing(1 if enable else 0))


def kernel_timing_read_split():
    """((FFMA kernels ms, launches), (tensor-core sum kernel ms, launches)) since kernel_timing(True)."""
    ms = (ctypes.c_double * 2)()
    cnt = (_i32 * 2)()
    check(load().pc_kernel_timing_read_split(ms, cnt))
    return (ms[0], cnt[0]), (ms[1], cnt[1])


def kernel_timing_read():
    """(summed main-kernel ms, launches) recorded since kernel_timing(True)."""
    ms, cnt = ctypes.c_double(), ctypes.c_int32()
    check(load().pc_kernel_timing_read(ctypes.byref(ms), ctypes.byref(cnt)))
    return ms.value, cnt.value


def microbench(kind: int):
    lib = load()
    rate, secs = ctypes.c_double(), ctypes.c_double()
    check(lib.pc_microbench(kind, ctypes.byref(rate), ctypes.byref(secs)))
    return rate.value, secs.value


# --- device memory (used by the lattice mirror; no torch dependency) --------

class DeviceBuffer:
    """A cudaMalloc'd, zero-filled buffer owned by Python."""

    def __init__(self, nbytes: int):
        self.nbytes = int(nbytes)
        ptr = ctypes.c_void_p()
        rc = load().pc_device_alloc(self.nbytes, ctypes.byref(ptr))
        if rc != PC_OK:
            raise MemoryError(f"cannot allocate {self.nbytes} device bytes: {last_error()}")
        self.ptr = ptr.value

    def to_host(self, dtype, count: int) -> np.ndarray:
        out = np.empty(count, dtype=dtype)
        lib = load()
        check(lib.pc_memcpy_d2h(out.ctypes.data, self.ptr, out.nbytes, None))
        check(lib.pc_stream_sync(None))
        return out

    def free(self) -> None:
        if getattr(self, "ptr", None):
            try:
                _handle.pc_device_free(self.ptr)
            finally:
                self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass
