"""Runs the C++ drop-in test binary (tests/cpp/test_dropin.cpp, built by __graft_entry__.build()
against the reference headers): pixelseg::gpu::X vs the reference's pixelseg::X, bit for bit."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

BIN = os.path.join(ROOT, "build", "test_dropin")


@pytest.mark.skipif(not os.path.exists(BIN), reason="build/test_dropin not built (needs /root/reference at build time)")
def test_cpp_dropin_matches_reference():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
