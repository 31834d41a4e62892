"""The C-ABI library loads on a CPU-only host and exports every symbol the
header declares, with the header's constants; no compute call is made."""

from __future__ import annotations

import ctypes
import re
import subprocess

import pytest

from paper_1901_11204_b200 import _lib
from tests.conftest import ROOT, _have_gpu

HEADER = (ROOT / "include" / "paircount.h").read_text()


def declared_functions():
    body = re.sub(r"/\*.*?\*/", "", HEADER, flags=re.S)
    return sorted(set(re.findall(r"\b(pc_[a-z0-9_]+)\s*\(", body)))


def test_header_and_binding_agree():
    assert declared_functions() == sorted(_lib.EXPORTED)


def test_library_exports_every_declared_symbol():
    lib = _lib.load(require_device=False)
    for name in declared_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r" T (pc_\w+)", out))
    assert set(declared_functions()) <= exported


def test_constants_match_header():
    defines = dict(re.findall(r"#define (PC_\w+) \(?(-?\d+)\)?", HEADER))
    for name, val in defines.items():
        assert getattr(_lib, name) == int(val), name


def test_struct_layouts():
    assert ctypes.sizeof(_lib.PairsResult) == 40
    assert ctypes.sizeof(_lib.LatticeResult) == 48


def test_pure_functions_without_device():
    lib = _lib.load(require_device=False)
    assert lib.pc_version().startswith(b"paircount-b200")
    assert lib.pc_lattice_grid_cells(512) == 1027**3
    assert lib.pc_lattice_key_bytes(512) == 4
    assert lib.pc_lattice_key_bytes(900) == 8
    assert _lib.workspace_bytes(1 << 20) >= 16 << 20


@pytest.mark.skipif(_have_gpu(), reason="checks the no-GPU failure mode")
def test_fails_loudly_without_device():
    with pytest.raises(_lib.PaircountUnavailable):
        _lib.pairs_host(__import__("numpy").zeros((4, 3), "f4"), _lib.PC_COLLISION, _lib.PC_BALANCED, [0, 4])
