"""Shared fixtures. `-m gpu` tests need a B200 and the built libgraft_cuda.so; everything else
runs on CPU (the oracle, the host-side mirror, the C-ABI symbol table, gloo multi-process)."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libgraft_cuda.so")


def load_golden(name):
    path = os.path.join(GOLDEN, name)
    if not os.path.exists(path):
        pytest.skip(f"golden fixture {name} not generated")
    return np.load(path)


@pytest.fixture(scope="session")
def glayers():
    return load_golden("layers.npz")


@pytest.fixture(scope="session")
def gnets():
    return load_golden("nets.npz")


def config_text(name):
    """Text of a proj/configs net (sk, sw, u, usk), from tests/golden/configs.npz."""
    return bytes(load_golden("configs.npz")[name.replace(".net", "")]).decode()


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint32 if a.dtype == np.float32 else np.uint64 if a.dtype == np.float64 else a.dtype)


def assert_bitwise(got, want, what=""):
    got = np.asarray(got)
    want = np.asarray(want)
    assert got.shape == want.shape, f"{what}: shape {got.shape} != {want.shape}"
    if not np.array_equal(bits(got), bits(want)):
        diff = np.flatnonzero(bits(got).ravel() != bits(want).ravel())
        i = diff[0]
        raise AssertionError(f"{what}: {diff.size} of {got.size} elements differ bitwise; first at "
                             f"{i}: got {got.ravel()[i]!r} want {want.ravel()[i]!r}")
