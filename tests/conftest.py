"""Shared fixtures.  `-m gpu` tests need a B200 (run under gpurun); the rest
run on the CPU-only dev container in a few minutes."""

from __future__ import annotations

import glob
import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu under gpurun")
    config.addinivalue_line("markers", "slow: long-running; still part of the default suites")


def _have_gpu() -> bool:
    return bool(glob.glob("/dev/nvidia[0-9]*"))


def pytest_collection_modifyitems(config, items):
    if _have_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container (run under gpurun)")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def golden_small():
    return json.loads((GOLDEN / "golden_small.json").read_text())


@pytest.fixture(scope="session")
def golden_configs():
    return json.loads((GOLDEN / "golden_configs.json").read_text())
