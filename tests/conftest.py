"""Shared test setup: the `gpu` marker, import paths and golden fixtures."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden")
for p in (REPO, os.path.join(REPO, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libartemis.so")


def load_golden(name: str):
    path = os.path.join(GOLDEN, name + ".npz")
    if not os.path.exists(path):
        pytest.skip(f"golden fixture {name}.npz absent")
    return np.load(path, allow_pickle=False)


@pytest.fixture(scope="session")
def golden_kernels():
    return load_golden("kernels")


@pytest.fixture(scope="session")
def golden_mini():
    return load_golden("scene_mini")


@pytest.fixture(scope="session")
def golden_scaled():
    return load_golden("scaled")


@pytest.fixture(scope="session")
def golden_c0():
    return load_golden("scene_c0")


@pytest.fixture(scope="session")
def golden_c2():
    return load_golden("scene_c2")


@pytest.fixture(scope="session")
def golden_backward():
    return load_golden("backward")


@pytest.fixture(scope="session")
def golden_post():
    return load_golden("post")


@pytest.fixture(scope="session")
def golden_asset():
    return load_golden("asset")


@pytest.fixture(scope="session")
def golden_fit():
    return load_golden("fit")
