"""Test helpers: rebuild golden inputs from their recipes and digest them."""

from __future__ import annotations

import hashlib

import numpy as np

from paper_1901_11204_b200 import generators as gen


def digest(arr: np.ndarray) -> str:
    """Same digest as tests/golden/make_golden.py."""
    arr = np.ascontiguousarray(arr)
    h = hashlib.sha256()
    h.update(str(arr.dtype).encode())
    h.update(str(arr.shape).encode())
    h.update(arr.tobytes())
    return h.hexdigest()


def spi_input(case: dict) -> np.ndarray:
    """The object array of a golden SPI case (regenerated or stored)."""
    if case.get("gen") is None:
        return np.asarray(case["points"], dtype=np.dtype(case["dtype"]))
    kind, n, box, seed, dtype = case["gen"]
    assert kind == "random_spheres"
    arr = gen.random_spheres(n, box, seed)
    return arr.astype(np.float32) if dtype == "float32" else arr


def lattice_input(case: dict) -> np.ndarray:
    if case.get("gen") is None:
        return np.asarray(case["beads"], dtype=np.int64).reshape(-1, 3)
    kind, *args = case["gen"]
    if kind == "random_chain":
        return gen.random_chain(*args)[0]
    return gen.normal_cloud(*args)


def config_input(golden_configs: dict, name: str) -> np.ndarray:
    """Inputs of the BASELINE configs."""
    if name == "cfg1_cloud":
        return gen.normal_cloud(*golden_configs["cfg1"]["cloud"]["args"])
    if name == "cfg1_chain":
        return gen.random_chain(*golden_configs["cfg1"]["chain"]["args"])[0]
    if name in ("cfg2", "cfg3", "cfg4u"):
        n, box, seed = golden_configs[name]["args"]
        return gen.random_spheres(n, box, seed).astype(np.float32)
    if name == "cfg4c":
        return gen.clustered_spheres(2**22).astype(np.float32)
    if name == "cfg5":
        return gen.grid_points(2**26)
    raise KeyError(name)
